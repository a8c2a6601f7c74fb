set -u
O=gpurun_out
mkdir -p $O
python -m paper_2409_17658_b200.build > $O/s19_build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "chain_every_power or split or tile64 or variant or stream_k or m8_every or power_sequence_matches" > $O/s19_pytest.log 2>&1
echo "pytest rc=$?"; tail -2 $O/s19_pytest.log
for rep in 1 2; do
echo "== before (RD_LIB=librd_ab.so)"; RD_LIB=$PWD/paper_2409_17658_b200/librd_ab.so timeout 600 python tools/alpha_cost_probe.py
echo "== after"; timeout 600 python tools/alpha_cost_probe.py
done > $O/s19_alpha_ab.txt 2>&1; cat $O/s19_alpha_ab.txt
