set -u
O=gpurun_out
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "tma_mainloop or tail_split or tunes_dpx or long_cp_async or stream_k or split_k or every_power" > $O/s32_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/s32_pytest.txt
timeout 900 python tools/tma_policy_probe.py 8:1 8:8 9:8 > $O/s32_tma_policy.txt 2>&1
for rep in 1 2; do
  timeout 300 python tools/ab_step.py 9 5
  timeout 300 python tools/ab_step.py 8 20
done > $O/s32_ab.txt 2>&1
tail -3 $O/s32_pytest.txt; cat $O/s32_tma_policy.txt $O/s32_ab.txt
