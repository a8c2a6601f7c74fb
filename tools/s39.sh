set -u
O=gpurun_out
mkdir -p $O
for rep in 1 2; do
  timeout 300 python tools/ab_step.py 7 20
  for v in librd.so librd_sku8.so librd_sku4.so librd_sksh0.so librd_sko2.so; do
    RD_LIB=$PWD/paper_2409_17658_b200/$v RD_STREAM_K=3 RD_TMA=0 timeout 300 python tools/ab_step.py 7 20
  done
done > $O/s39_sk_variants.txt 2>&1; cat $O/s39_sk_variants.txt
