set -u
O=gpurun_out
mkdir -p $O
timeout 300 python __graft_entry__.py > $O/s54_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "every_power or tail_split or tunes_dpx or small" > $O/s54_pytest.txt 2>&1; echo "pytest rc=$?"; tail -2 $O/s54_pytest.txt
timeout 300 python tools/ab_step.py 9 5
