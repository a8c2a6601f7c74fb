set -u
O=gpurun_out
mkdir -p $O
python tools/small_profile.py 3 > $O/s53_plain.log 2>&1 && \
timeout 300 ncu --set full --clock-control none --import-source on -k regex:small_chain --launch-skip 1 --launch-count 1 -o $O/s53_small3 python tools/small_profile.py 3 > $O/s53_ncu.log 2>&1
echo rc=$?
