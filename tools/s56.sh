set -u
O=gpurun_out
mkdir -p $O
for rep in 1 2; do
  for v in librd.so librd_t64o0.so librd_t64o1.so librd_t64o5.so; do
    RD_LIB=$PWD/paper_2409_17658_b200/$v timeout 300 python tools/ab_step.py 7 20
  done
done > $O/s56_t64_order.txt 2>&1; cat $O/s56_t64_order.txt
