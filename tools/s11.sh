set -u
O=gpurun_out
mkdir -p $O
python -m paper_2409_17658_b200.build > $O/s11_build.log 2>&1; echo "build rc=$?"
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "panel_stats or allgather" > $O/s11_pytest.log 2>&1
echo "pytest rc=$?"; tail -2 $O/s11_pytest.log
timeout 300 python tools/time_panel_stats.py 0 1 2 4 10 16 > $O/s11_panel_stats.txt 2>&1; cat $O/s11_panel_stats.txt
timeout 600 ncu --set full --clock-control none -k regex:panel_stats -s 2 -c 1 -o $O/s11_panel_stats python tools/time_panel_stats.py 10 > $O/s11_ncu_ps.log 2>&1; echo "ncu rc=$?"
