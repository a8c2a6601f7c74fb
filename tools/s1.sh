set -u
O=gpurun_out
mkdir -p $O
python -m paper_2409_17658_b200.build > $O/s1_build.log 2>&1; echo "build rc=$?"
timeout 2700 python -m pytest tests -m gpu -q -x --durations=25 > $O/s1_pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -30 $O/s1_pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --ttp-structured-only-m > $O/s1_bench.json 2> $O/s1_bench.err
echo "bench rc=$?"; cat $O/s1_bench.json | head -c 6000
