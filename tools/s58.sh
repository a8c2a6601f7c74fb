set -u
O=gpurun_out
mkdir -p $O
timeout 1200 python tools/wave_probe.py > $O/s58_wave.txt 2>&1; cat $O/s58_wave.txt
