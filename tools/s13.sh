set -u
O=gpurun_out
mkdir -p $O
python -m paper_2409_17658_b200.build > $O/s13_build.log 2>&1; echo "build rc=$?"
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "small_chain or power_sequence_matches or table2" > $O/s13_pytest.log 2>&1
echo "pytest rc=$?"; tail -2 $O/s13_pytest.log
timeout 300 python tools/small_m_latency.py 1 3 4 5 6 > $O/s13_small.txt 2>&1; cat $O/s13_small.txt
timeout 120 tools/hadd_probe > $O/s13_hadd_probe.txt 2>&1; cat $O/s13_hadd_probe.txt
timeout 900 python tools/hash_repro.py 1 3 > $O/s13_hash.txt 2>&1; cat $O/s13_hash.txt | cut -c1-300
