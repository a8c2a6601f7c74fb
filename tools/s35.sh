set -u
O=gpurun_out
mkdir -p $O
for rep in 1 2; do
  for v in librd.so librd_et1.so; do
    RD_LIB=$PWD/paper_2409_17658_b200/$v RD_TMA=2 RD_TILE=128 timeout 300 python tools/ab_step.py 7 20
    RD_LIB=$PWD/paper_2409_17658_b200/$v RD_TMA=2 RD_TILE=128 RD_VARIANT=3 timeout 300 python tools/ab_step.py 8 20
    RD_LIB=$PWD/paper_2409_17658_b200/$v RD_VARIANT=4 timeout 300 python tools/ab_step.py 8 20
  done
done > $O/s35_epi_tma_m7.txt 2>&1
cat $O/s35_epi_tma_m7.txt
