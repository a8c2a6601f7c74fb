set -u
O=gpurun_out
mkdir -p $O
python -m paper_2409_17658_b200.build > $O/s8_build.log 2>&1; echo "build rc=$?"
timeout 1500 python tools/hash_repro.py 1,3,0 2 > $O/s8_hash.txt 2>&1; echo "hash rc=$?"; cat $O/s8_hash.txt | cut -c1-600
timeout 300 python tools/refill_probe.py > $O/s8_refill.txt 2>&1; cat $O/s8_refill.txt
