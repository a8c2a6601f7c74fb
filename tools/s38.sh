set -u
O=gpurun_out
mkdir -p $O
python tools/m7_profile.py skfull 7 > /dev/null 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:minplus_gemm --launch-skip 4 --launch-count 1 -o $O/s38_m7_skfull python tools/m7_profile.py skfull 7 > $O/s38_full.log 2>&1
echo rc=$?
