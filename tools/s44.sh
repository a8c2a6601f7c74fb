set -u
O=gpurun_out
mkdir -p $O
for rep in 1 2; do
  for v in librd_or2.so librd_or4.so librd_or5.so; do
    RD_VARIANT=3 RD_LIB=$PWD/paper_2409_17658_b200/$v timeout 300 python tools/ab_step.py 9 5
  done
  RD_VARIANT=4 RD_LIB=$PWD/paper_2409_17658_b200/librd_or5.so timeout 300 python tools/ab_step.py 9 5
done > $O/s44_order45_ab.txt 2>&1; cat $O/s44_order45_ab.txt
