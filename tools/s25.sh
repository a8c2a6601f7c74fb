set -u
O=gpurun_out
mkdir -p $O
for c in plain tail2 s4; do
  timeout 300 ncu --clock-control none -k regex:minplus_gemm --launch-skip 4 --launch-count 1 \
    --metrics gpu__time_duration.sum,sm__cycles_active.avg,sm__cycles_active.max,sm__cycles_active.min,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__waves_per_multiprocessor,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__occupancy_limit_registers,launch__occupancy_limit_shared_mem,sm__cycles_elapsed.max,dram__bytes_read.sum,lts__t_bytes.sum \
    --csv python tools/m7_profile.py $c > $O/s25_$c.csv 2>&1
done
timeout 300 ncu --set full --clock-control none -k regex:minplus_gemm --launch-skip 4 --launch-count 1 -o $O/s25_m7_plain python tools/m7_profile.py plain > $O/s25_full.log 2>&1
for c in plain tail2 s4; do echo "== $c"; grep -v "^==PROF==" $O/s25_$c.csv | tail -16; done
