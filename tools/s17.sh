set -u
O=gpurun_out
mkdir -p $O
python -m paper_2409_17658_b200.build > $O/s17_build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "chain_every_power or split or tile64 or variant or tunes or m8_every" > $O/s17_pytest.log 2>&1
echo "pytest rc=$?"; tail -2 $O/s17_pytest.log
timeout 600 python tools/alpha_cost_probe.py > $O/s17_alpha.txt 2>&1; cat $O/s17_alpha.txt
