set -u
O=gpurun_out
mkdir -p $O
for rep in 1 2; do
  RD_VARIANT=3 timeout 300 python tools/ab_step.py 9 5
  RD_VARIANT=2 RD_LIB=$PWD/paper_2409_17658_b200/librd_or2.so timeout 300 python tools/ab_step.py 9 5
  RD_VARIANT=2 timeout 300 python tools/ab_step.py 9 5
done > $O/s57_d2.txt 2>&1; cat $O/s57_d2.txt
