set -u
O=gpurun_out
mkdir -p $O
python -m paper_2409_17658_b200.build > $O/s9_build.log 2>&1; echo "build rc=$?"
timeout 2400 python -m pytest tests -m gpu -q -x --durations=10 > $O/s9_pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -4 $O/s9_pytest_gpu.log
timeout 300 python tools/time_panel_stats.py 0 1 2 4 10 16 > $O/s9_panel_stats.txt 2>&1; cat $O/s9_panel_stats.txt
timeout 600 python tools/wave_probe.py 6:1 7:1 7:2 8:8 > $O/s9_wave.txt 2>&1; cut -c1-160 $O/s9_wave.txt
# the peer all-gather form's right-operand traffic on one GPU (what would cross NVLink at N > 1)
timeout 900 ncu --metrics gpu__time_duration.sum,l1tex__m_xbar2l1tex_read_bytes_mem_global_op_ldgsts_cache_access.sum,l1tex__m_xbar2l1tex_read_bytes.sum,lts__t_bytes.sum,dram__bytes_read.sum --clock-control none -k regex:minplus_gemm -s 3 -c 1 --csv python bench.py --form peer --steps 2 --warmup 2 --no-e2e --no-cpu-baseline > $O/s9_peer_ncu.csv 2>&1
echo "peer ncu rc=$?"; grep minplus $O/s9_peer_ncu.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
timeout 900 ncu --metrics gpu__time_duration.sum,l1tex__m_xbar2l1tex_read_bytes.sum,lts__t_bytes.sum,dram__bytes_read.sum --clock-control none -k regex:minplus_gemm -s 3 -c 1 --csv python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu-baseline > $O/s9_repl_ncu.csv 2>&1
echo "repl ncu rc=$?"; grep minplus $O/s9_repl_ncu.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
