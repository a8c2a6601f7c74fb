set -u
O=gpurun_out
mkdir -p $O
python -m paper_2409_17658_b200.build > $O/s12_build.log 2>&1; echo "build rc=$?"
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "small_chain or power_sequence_matches or table2 or border" > $O/s12_pytest.log 2>&1
echo "pytest rc=$?"; tail -2 $O/s12_pytest.log
timeout 300 python tools/small_m_latency.py 1 2 3 4 5 6 > $O/s12_small.txt 2>&1; cat $O/s12_small.txt
