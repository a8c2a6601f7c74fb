set -u
O=gpurun_out
mkdir -p $O
for rep in 1 2 3; do
  for v in librd.so librd_m32o2.so; do
    RD_LIB=$PWD/paper_2409_17658_b200/$v timeout 300 python tools/mul32_probe.py 7411
  done
done > $O/s47_mul32_ab.txt 2>&1; cat $O/s47_mul32_ab.txt
