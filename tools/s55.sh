set -u
O=gpurun_out
mkdir -p $O
timeout 600 python tools/ab_step.py 10 3 > $O/s55_m10.txt 2>&1; cat $O/s55_m10.txt
