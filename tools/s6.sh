set -u
O=gpurun_out
mkdir -p $O
python -m paper_2409_17658_b200.build > $O/s6_build.log 2>&1; echo "build rc=$?"
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "panel_stats or variant" > $O/s6_pytest.log 2>&1
echo "pytest rc=$?"; tail -3 $O/s6_pytest.log
timeout 300 python tools/time_panel_stats.py > $O/s6_panel_stats.txt 2>&1; cat $O/s6_panel_stats.txt
timeout 900 python tools/variant_tma_probe.py > $O/s6_variants.txt 2>&1; cat $O/s6_variants.txt
cat > /tmp/m7.py <<'PY'
import sys; sys.path.insert(0, ".")
import torch, paper_2409_17658_b200 as rd
tn, split = int(sys.argv[1]), int(sys.argv[2])
rd.rd_set_gemm_tile(tn); rd.rd_set_split_k(bool(split))
ch = rd.Chain(7, alpha_max=10)
for _ in range(6): ch.step()
torch.cuda.synchronize()
PY
for cfg in "128 0" "64 1"; do
timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,sm__cycles_elapsed.avg,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv python /tmp/m7.py $cfg > $O/s6_m7_ncu.csv 2>&1
echo "== $cfg"; grep -E "minplus|combine" $O/s6_m7_ncu.csv | tail -10 | awk -F'","' '{print $5" | "$(NF-2)" "$NF}' | cut -c1-60,200-320
done
