"""Time-to-periodicity of the C loop (rd_power_sequence_timed) vs the Python driver, per m and
method, repeated (first call includes one-time costs such as the slab layout build)."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2409_17658_b200 as rd  # noqa: E402
from paper_2409_17658_b200 import dist as D  # noqa: E402

torch.cuda.init()
ms = [int(x) for x in sys.argv[1:]] or [8, 9]
for m in ms:
    for method in (1, 0):
        for rep in range(3 if method == 1 else 2):
            t0 = time.perf_counter()
            r = rd.rd_power_sequence(m, 50, 10, method=method)
            tw = time.perf_counter() - t0
            rp = D.power_sequence(m, 50, 10, method=method)
            print(f"m={m} method={method} rep={rep} C: build {r['t_build']*1e3:.1f} chain {r['t_chain']*1e3:.1f} "
                  f"wall {tw*1e3:.1f} ms | py: build {rp['t_build']*1e3:.1f} chain {rp['t_chain']*1e3:.1f} ms",
                  flush=True)
