set -u
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "tunes_dpx or long_cp_async or tail_split or variant" > $O/s28_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/s28_pytest.txt
for rep in 1 2 3; do
  for v in auto 3 4; do
    if [ $v = auto ]; then timeout 300 python tools/ab_step.py 8 20; else RD_VARIANT=$v timeout 300 python tools/ab_step.py 8 20; fi
  done
done > $O/s28_m8_dpx.txt 2>&1
tail -3 $O/s28_pytest.txt; cat $O/s28_m8_dpx.txt
