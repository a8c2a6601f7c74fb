set -u
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "tma_mainloop or tunes_dpx or long_cp_async or every_power" > $O/s45_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/s45_pytest.txt
for rep in 1 2; do
  timeout 300 python tools/ab_step.py 9 5
  for v in librd.so librd_cp2.so; do
    RD_LIB=$PWD/paper_2409_17658_b200/$v timeout 300 python tools/ab_step.py 7 20
    RD_LIB=$PWD/paper_2409_17658_b200/$v timeout 300 python tools/ab_step.py 6 20
  done
  for v in librd.so librd_cp2s.so; do
    RD_LIB=$PWD/paper_2409_17658_b200/$v RD_TMA=0 RD_VARIANT=3 timeout 300 python tools/ab_step.py 8 20
  done
done > $O/s45_cp_order_ab.txt 2>&1
tail -3 $O/s45_pytest.txt; cat $O/s45_cp_order_ab.txt
