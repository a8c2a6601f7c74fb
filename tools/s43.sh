set -u
O=gpurun_out
mkdir -p $O
for rep in 1 2; do
  for d in 4 3; do
    for v in librd.so librd_or2.so librd_or3.so; do
      RD_VARIANT=$d RD_LIB=$PWD/paper_2409_17658_b200/$v timeout 300 python tools/ab_step.py 9 5
    done
  done
done > $O/s43_order23_ab.txt 2>&1; cat $O/s43_order23_ab.txt
