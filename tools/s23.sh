set -u
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "stream_k or split_k or tile64 or variants or every_power" > $O/s23_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/s23_pytest.txt
timeout 600 python tools/sk_probe.py 6:1 7:1 7:2 7:4 8:1 8:8 > $O/s23_sk_probe.txt 2>&1
for rep in 1 2 3; do
  for m in 8 7; do
    for v in librd.so librd_sh0c.so; do
      RD_LIB=$PWD/paper_2409_17658_b200/$v timeout 300 python tools/ab_step.py $m 20
    done
  done
done > $O/s23_shift_cp_ab.txt 2>&1
tail -3 $O/s23_pytest.txt; cat $O/s23_sk_probe.txt $O/s23_shift_cp_ab.txt
