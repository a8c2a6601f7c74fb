set -u
O=gpurun_out
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "tma_mainloop or tunes_dpx or long_cp_async or v24 or m8_full" > $O/s42_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/s42_pytest.txt
for rep in 1 2; do
  for v in librd.so librd_sp0.so; do
    RD_LIB=$PWD/paper_2409_17658_b200/$v timeout 300 python tools/ab_step.py 9 5
    RD_LIB=$PWD/paper_2409_17658_b200/$v timeout 300 python tools/ab_step.py 8 20
  done
done > $O/s42_split_ab.txt 2>&1
tail -3 $O/s42_pytest.txt; cat $O/s42_split_ab.txt
