set -u
O=gpurun_out
mkdir -p $O
python -m paper_2409_17658_b200.build > $O/s15_build.log 2>&1; echo "build rc=$?"
timeout 600 python tools/refill_probe.py 9 dephase > $O/s15_dephase9.txt 2>&1; cat $O/s15_dephase9.txt
timeout 600 python tools/refill_probe.py 8 dephase > $O/s15_dephase8.txt 2>&1; cat $O/s15_dephase8.txt
