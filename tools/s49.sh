set -u
O=gpurun_out
mkdir -p $O
for rep in 1 2; do
  timeout 300 python tools/ab_step.py 8 20
  RD_VARIANT=3 timeout 300 python tools/ab_step.py 8 20
  RD_VARIANT=4 timeout 300 python tools/ab_step.py 8 20
done > $O/s49_m8_d.txt 2>&1
timeout 600 python tools/tma_policy_probe.py 8:8 9:8 >> $O/s49_m8_d.txt 2>&1
cat $O/s49_m8_d.txt
