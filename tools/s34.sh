set -u
O=gpurun_out
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "tma_mainloop or tail_split or tunes_dpx or long_cp_async or every_power or m8_full or stream_k or peer or panel" > $O/s34_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/s34_pytest.txt
for rep in 1 2; do
  for v in librd.so librd_et0.so; do
    RD_LIB=$PWD/paper_2409_17658_b200/$v timeout 300 python tools/ab_step.py 9 5
    RD_LIB=$PWD/paper_2409_17658_b200/$v timeout 300 python tools/ab_step.py 8 20
    RD_LIB=$PWD/paper_2409_17658_b200/$v RD_TMA=2 timeout 300 python tools/ab_step.py 7 20
  done
done > $O/s34_epi_tma_ab.txt 2>&1
tail -3 $O/s34_pytest.txt; cat $O/s34_epi_tma_ab.txt
