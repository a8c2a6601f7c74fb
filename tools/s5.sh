set -u
O=gpurun_out
mkdir -p $O
python -m paper_2409_17658_b200.build > $O/s5_build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "panel_stats or allgather or tile64 or variant" > $O/s5_pytest.log 2>&1
echo "pytest rc=$?"; tail -3 $O/s5_pytest.log
timeout 300 python tools/time_panel_stats.py > $O/s5_panel_stats.txt 2>&1; cat $O/s5_panel_stats.txt
timeout 900 python tools/sk_probe.py > $O/s5_sk_probe.txt 2>&1; echo "probe rc=$?"; cat $O/s5_sk_probe.txt
