set -u
O=gpurun_out
mkdir -p $O
for rep in 1 2; do
  for v in librd.so librd_or8.so librd_or9.so librd_or10.so; do
    RD_VARIANT=3 RD_LIB=$PWD/paper_2409_17658_b200/$v timeout 300 python tools/ab_step.py 9 5
  done
done > $O/s52_order8910.txt 2>&1; cat $O/s52_order8910.txt
