"""TMA mainloop vs cp.async mainloop for the dense chain step: identical powers and stats,
and the median step time (CUDA events), per order."""
import statistics
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2409_17658_b200 as rd  # noqa: E402
from paper_2409_17658_b200 import dist as D  # noqa: E402


def run(m, tma, r0=0, r1=None, steps=6, reps=6):
    rd.rd_set_gemm_tma(tma)
    st = torch.cuda.current_stream()
    ch = rd.Chain(m, alpha_max=10, row_begin=r0, row_end=r1, stream=st)
    stats = []
    for _ in range(steps):
        stats.append(ch.step().cpu().numpy().copy())
    rows = ch.read_rows(ch.k)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record(st); ch.step(); b.record(st)
    torch.cuda.synchronize()
    ch.close()
    rd.rd_set_gemm_tma(1)
    return np.stack(stats), rows, statistics.median(a.elapsed_time(b) for a, b in ev)


for m, parts in ((5, 1), (6, 1), (7, 1), (8, 1), (8, 8), (9, 1)):
    N = rd.count_words(m)
    r0, r1 = D.panel_bounds(N, parts, 0)
    s0, x0, t0 = run(m, False, r0, r1, reps=3 if m == 9 else 6)
    s1, x1, t1 = run(m, True, r0, r1, reps=3 if m == 9 else 6)
    print(f"m={m} rows=[{r0},{r1}) identical={bool((s0 == s1).all() and (x0 == x1).all())}  "
          f"cp.async {t0:.3f} ms  TMA {t1:.3f} ms  ({t0 / t1:.4f}x)", flush=True)
