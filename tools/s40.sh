set -u
O=gpurun_out
mkdir -p $O
for rep in 1 2; do
  RD_VARIANT=3 timeout 300 python tools/ab_step.py 9 5
  RD_VARIANT=4 timeout 300 python tools/ab_step.py 9 5
  RD_LIB=$PWD/paper_2409_17658_b200/librd_d5.so RD_VARIANT=8 timeout 300 python tools/ab_step.py 9 5
  RD_LIB=$PWD/paper_2409_17658_b200/librd_d6.so RD_VARIANT=8 timeout 300 python tools/ab_step.py 9 5
done > $O/s40_d56.txt 2>&1; cat $O/s40_d56.txt
