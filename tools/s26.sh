set -u
O=gpurun_out
mkdir -p $O
for rep in 1 2 3 4; do
  for v in librd.so librd_op0.so; do
    RD_LIB=$PWD/paper_2409_17658_b200/$v timeout 300 python tools/ab_step.py 9 5
  done
done > $O/s26_epi_opaque_ab.txt 2>&1; cat $O/s26_epi_opaque_ab.txt
