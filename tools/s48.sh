set -u
O=gpurun_out
mkdir -p $O
for rep in 1 2; do
  for v in librd.so librd_sh0.so librd_sh2.so librd_sh3.so; do
    RD_VARIANT=3 RD_LIB=$PWD/paper_2409_17658_b200/$v timeout 300 python tools/ab_step.py 9 5
  done
done > $O/s48_shift_order2.txt 2>&1; cat $O/s48_shift_order2.txt
