set -u
O=gpurun_out
mkdir -p $O
timeout 1200 python tools/tma_policy_probe.py > $O/s31_tma_policy.txt 2>&1
cat $O/s31_tma_policy.txt
