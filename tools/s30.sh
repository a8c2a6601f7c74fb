set -u
O=gpurun_out
mkdir -p $O
for rep in 1 2; do
  timeout 300 python tools/ab_step.py 8 20
  RD_TMA=2 timeout 300 python tools/ab_step.py 8 20
  RD_TMA=2 RD_SPLIT_K=0 timeout 300 python tools/ab_step.py 8 20
  RD_SPLIT_K=0 timeout 300 python tools/ab_step.py 8 20
  RD_TMA=2 timeout 300 python tools/ab_step.py 7 20
done > $O/s30_tma_m8.txt 2>&1
cat $O/s30_tma_m8.txt
