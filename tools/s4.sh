set -u
O=gpurun_out
mkdir -p $O
python -m paper_2409_17658_b200.build > $O/s4_build.log 2>&1; echo "build rc=$?"
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "panel_stats or allgather" > $O/s4_pytest.log 2>&1
echo "pytest rc=$?"; tail -3 $O/s4_pytest.log
timeout 300 python tools/time_panel_stats.py > $O/s4_panel_stats.txt 2>&1; cat $O/s4_panel_stats.txt
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv -k regex:panel_stats -c 3 python tools/time_panel_stats.py > $O/s4_ps_ncu.csv 2>&1; grep panel_stats $O/s4_ps_ncu.csv | tail -4 | cut -c1-100,240-400
RD_DIST_BACKEND=gloo RD_FORCE_DEVICE=0 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 tools/next2_ranks.py $O/s4_next2_ranks.json > $O/s4_next2.log 2>&1
echo "next2 rc=$?"; tail -5 $O/s4_next2.log | cut -c1-600
