"""Small-order latency: Algorithm 2 end to end through the C loop (rd_power_sequence, speculative
depth) vs the Python row-panel driver, wall clock, warm (best of 5).  (The CPU oracle's own
time to periodicity is reported by bench.py's cpu_baseline leg, the one place outside tests
that runs it.)"""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2409_17658_b200 as rd  # noqa: E402
from paper_2409_17658_b200 import dist as D  # noqa: E402

torch.cuda.init()
for m in [int(x) for x in sys.argv[1:]] or [3, 4, 5, 6, 7]:
    for method in (0, 1):
        best = 1e9
        for _ in range(5):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = rd.rd_power_sequence(m, 50, 10, method=method)
            best = min(best, time.perf_counter() - t0)
        rp = None
        for _ in range(3):
            rp = D.power_sequence(m, 50, 10, method=method)
        print(f"m={m} method={method} C-loop {best*1e3:.3f} ms  py-driver build {rp['t_build']*1e3:.3f} "
              f"chain {rp['t_chain']*1e3:.3f} ms  triple {(r['n0'], r['alpha'], r['beta'])}", flush=True)
