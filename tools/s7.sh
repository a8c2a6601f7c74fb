set -u
O=gpurun_out
mkdir -p $O
python -m paper_2409_17658_b200.build > $O/s7_build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "split or tile64 or stream_k or chain_every_power or panel" > $O/s7_pytest.log 2>&1
echo "pytest rc=$?"; tail -3 $O/s7_pytest.log
timeout 1200 python tools/wave_probe.py > $O/s7_wave.txt 2>&1; echo "probe rc=$?"; cat $O/s7_wave.txt
