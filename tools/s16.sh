set -u
O=gpurun_out
mkdir -p $O
python -m paper_2409_17658_b200.build > $O/s16_build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tunes or variant or power_sequence_m9" > $O/s16_pytest.log 2>&1
echo "pytest rc=$?"; tail -2 $O/s16_pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/s16_bench.json 2> $O/s16_bench.err
python -c "
import json; d=json.loads(open('$O/s16_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['dpx_cols'])"
