#!/bin/bash
# One GPU session: bench (both arms), ncu launch list, ncu --set full of the GEMM.
# usage: tools/gpu_round.sh <tag>   (outputs under gpurun_out/<tag>_*)
set -u
TAG=${1:-r01}
O=gpurun_out
mkdir -p $O
python -m paper_2409_17658_b200.build > $O/${TAG}_build.log 2>&1
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > $O/${TAG}_pytest_gpu.log 2>&1
  echo "pytest rc=$?"; tail -3 $O/${TAG}_pytest_gpu.log
  timeout 300 python __graft_entry__.py > $O/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
fi
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > $O/${TAG}_clocks.csv &
SMI=$!
python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
echo "bench rc=$?"
kill $SMI
python bench.py --impl reference --steps 3 --warmup 1 > $O/${TAG}_bench_ref.json 2> $O/${TAG}_bench_ref.err
echo "ref rc=$?"
CMD="python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > $O/${TAG}_plain.log 2>&1 &&
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches.csv $CMD > $O/${TAG}_ncu_launches.log 2>&1
echo "launches rc=$?"
$CMD > $O/${TAG}_plain2.log 2>&1 &&
# launch 7 = the power A^9, after the chain's DPX tuning (A^4..A^7) has chosen its mix
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:minplus_gemm -s 7 -c 1 -o $O/${TAG}_gemm $CMD > $O/${TAG}_ncu_full.log 2>&1
echo "full rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:panel_stats -s 2 -c 1 -o $O/${TAG}_panel_stats python tools/time_panel_stats.py > $O/${TAG}_ncu_ps.log 2>&1
echo "ps full rc=$?"
timeout 1200 python tools/wave_probe.py > $O/${TAG}_wave.txt 2>&1; echo "wave rc=$?"
timeout 300 python tools/alpha_cost_probe.py > $O/${TAG}_alpha_cost.txt 2>&1; cat $O/${TAG}_alpha_cost.txt
timeout 900 python tools/hash_repro.py 1 2 > $O/${TAG}_hash.txt 2>&1; cat $O/${TAG}_hash.txt
cat $O/${TAG}_bench.json; cat $O/${TAG}_bench_ref.json
