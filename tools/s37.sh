set -u
O=gpurun_out
mkdir -p $O
M="gpu__time_duration.sum,sm__cycles_active.avg,sm__cycles_active.max,sm__cycles_active.min,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__waves_per_multiprocessor,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__occupancy_limit_registers,launch__occupancy_limit_shared_mem,sm__cycles_elapsed.max,dram__bytes_read.sum,lts__t_bytes.sum,smsp__inst_executed.sum,launch__occupancy_per_block_size,sm__maximum_warps_per_active_cycle_pct"
for c in plain skfull skhyb; do
  python tools/m7_profile.py $c 7 > /dev/null 2>&1 && \
  timeout 300 ncu --clock-control none -k regex:minplus_gemm --launch-skip 4 --launch-count 1 --metrics $M --csv python tools/m7_profile.py $c 7 > $O/s37_$c.csv 2>&1
done
for c in plain skfull skhyb; do echo "== $c"; grep -v "^==" $O/s37_$c.csv | awk -F'","' '{print $(NF-2), $NF}' | tail -17; done
