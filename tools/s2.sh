set -u
O=gpurun_out
mkdir -p $O
python -m paper_2409_17658_b200.build > $O/s2_build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "small_chain or panel_stats or stream_k or power_sequence_matches or table2" > $O/s2_pytest.log 2>&1
echo "pytest rc=$?"; tail -5 $O/s2_pytest.log
timeout 600 python tools/sk_probe.py > $O/s2_sk_probe.txt 2>&1; echo "probe rc=$?"; cat $O/s2_sk_probe.txt
timeout 300 python tools/time_panel_stats.py > $O/s2_panel_stats.txt 2>&1; cat $O/s2_panel_stats.txt
timeout 300 python tools/small_m_latency.py > $O/s2_small.txt 2>&1; cat $O/s2_small.txt
