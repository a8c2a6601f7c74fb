set -u
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "tunes_dpx or long_cp_async or tma_mainloop" > $O/s50_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/s50_pytest.txt
for rep in 1 2 3; do
  timeout 300 python tools/ab_step.py 8 20
done > $O/s50_m8_tune.txt 2>&1
tail -3 $O/s50_pytest.txt; cat $O/s50_m8_tune.txt
