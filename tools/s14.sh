set -u
O=gpurun_out
mkdir -p $O
python -m paper_2409_17658_b200.build > $O/s14_build.log 2>&1; echo "build rc=$?"
timeout 120 tools/hadd_probe > $O/s14_hadd_probe.txt 2>&1; tail -3 $O/s14_hadd_probe.txt
# the N = 2 default bench path end to end (two ranks sharing cuda:0 over gloo: functional only)
RD_DIST_BACKEND=gloo RD_FORCE_DEVICE=0 timeout 1500 python bench.py --gpus 2 --steps 3 --warmup 3 > $O/s14_bench2.json 2> $O/s14_bench2.err
echo "bench2 rc=$?"; python -c "
import json; d=json.loads(open('$O/s14_bench2.json').read().strip().splitlines()[-1])
print({k: d[k] for k in ('n_gpus','value','ms_per_step')}, d['config'].get('detected'), {m: v.get('triple') for m, v in d['time_to_periodicity'].items()})"
tail -3 $O/s14_bench2.err
