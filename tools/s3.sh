set -u
O=gpurun_out
mkdir -p $O
python -m paper_2409_17658_b200.build > $O/s3_build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "small_chain or panel_stats or stream_k or power_sequence_matches or table2 or split_k" > $O/s3_pytest.log 2>&1
echo "pytest rc=$?"; tail -5 $O/s3_pytest.log
timeout 300 python tools/time_panel_stats.py > $O/s3_panel_stats.txt 2>&1; cat $O/s3_panel_stats.txt
timeout 300 python tools/small_m_latency.py 3 4 5 6 > $O/s3_small.txt 2>&1; cat $O/s3_small.txt
cat > /tmp/sk7.py <<'PY'
import sys; sys.path.insert(0, ".")
import torch, paper_2409_17658_b200 as rd
rd.rd_set_split_k(False); rd.rd_set_stream_k(int(sys.argv[1]))
ch = rd.Chain(7, alpha_max=10)
for _ in range(6): ch.step()
torch.cuda.synchronize()
PY
for mode in 0 2; do
timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv python /tmp/sk7.py $mode > $O/s3_sk7_ncu_$mode.csv 2>&1
grep -E "minplus_gemm|combine" $O/s3_sk7_ncu_$mode.csv | tail -6 | cut -c1-400
done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv -k regex:panel_stats python tools/time_panel_stats.py > $O/s3_ps_ncu.csv 2>&1; tail -4 $O/s3_ps_ncu.csv | cut -c1-300
