set -u
O=gpurun_out
mkdir -p $O
echo skip-build
for rep in 1 2 3; do
  for v in librd.so librd_sh1.so librd_sh2.so librd_sh4.so librd_sh5.so librd_sh7.so; do
    RD_LIB=$PWD/paper_2409_17658_b200/$v timeout 300 python tools/ab_step.py 9 5
  done
done > $O/s22_shift_ab.txt 2>&1; cat $O/s22_shift_ab.txt
