set -u
O=gpurun_out
mkdir -p $O
for rep in 1 2 3; do
  for m in 8 7; do
    for v in librd.so librd_fa1.so; do
      RD_LIB=$PWD/paper_2409_17658_b200/$v timeout 300 python tools/ab_step.py $m 20
    done
  done
done > $O/s27_epi_fastall_ab.txt 2>&1; cat $O/s27_epi_fastall_ab.txt
