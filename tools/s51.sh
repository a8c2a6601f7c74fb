set -u
O=gpurun_out
mkdir -p $O
for rep in 1 2; do
  for v in librd.so librd_u8.so librd_u4.so; do
    RD_VARIANT=3 RD_LIB=$PWD/paper_2409_17658_b200/$v timeout 300 python tools/ab_step.py 9 5
  done
done > $O/s51_unroll_order2.txt 2>&1; cat $O/s51_unroll_order2.txt
