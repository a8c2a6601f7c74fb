"""Small-order latency: Algorithm 2 to first detection through rd_power_sequence (dense:
the device-resident kernel of rd_small.cu, and with rd_set_small_chain(0) the host-driven
chain; structured), build and chain seconds as the library reports them, best of 5 warm runs.
(The CPU oracle's own time to periodicity is reported by bench.py's cpu_baseline leg.)"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2409_17658_b200 as rd  # noqa: E402

torch.cuda.init()
for m in [int(x) for x in sys.argv[1:]] or [3, 4, 5, 6, 7]:
    for label, method, small in (("dense device-resident", 0, True), ("dense host-driven", 0, False),
                                 ("structured", 1, True)):
        rd.rd_set_small_chain(small)
        runs = [rd.rd_power_sequence(m, 50, 10, method=method) for _ in range(6)][1:]
        rd.rd_set_small_chain(True)
        b = min(r["t_build"] for r in runs) * 1e3
        c = min(r["t_chain"] for r in runs) * 1e3
        r = runs[-1]
        print(f"m={m} {label:22s} build {b:.3f} ms  chain {c:.3f} ms  triple {(r['n0'], r['alpha'], r['beta'])} "
              f"k_stop {r['k_stop']}", flush=True)
