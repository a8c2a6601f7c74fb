set -u
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "tail_split or stream_k or split_k" > $O/s24_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/s24_pytest.txt
timeout 900 python tools/wave_probe.py > $O/s24_wave.txt 2>&1
tail -3 $O/s24_pytest.txt; cat $O/s24_wave.txt
