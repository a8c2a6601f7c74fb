set -u
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "small" > $O/s36_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/s36_pytest.txt
timeout 600 python tools/small_m_latency.py 3 4 5 6 > $O/s36_small.txt 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/s36_bench.json 2> $O/s36_bench.err
python - <<'P' >> $O/s36_small.txt
import json
d = json.load(open("gpurun_out/s36_bench.json"))
print({k: (v.get("build_s"), v.get("chain_s"), v.get("total_s")) for k, v in d["time_to_periodicity"].items()})
P
tail -3 $O/s36_pytest.txt; cat $O/s36_small.txt
