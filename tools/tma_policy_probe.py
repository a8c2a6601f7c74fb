"""Dense chain step time (median of 10, CUDA events; the wave model's plan) per order / row
panel with the TMA mainloop policy of rd_set_gemm_tma 1 (TMA only for unsplit steps of >= 128
k-stages) against 2 (TMA for every 128-wide step, any split form): DESIGN.md §5."""
import statistics
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2409_17658_b200 as rd  # noqa: E402
from paper_2409_17658_b200 import dist as D  # noqa: E402


def med(m, r0, r1, reps=10):
    st = torch.cuda.current_stream()
    ch = rd.Chain(m, alpha_max=10, row_begin=r0, row_end=r1, stream=st)
    for _ in range(6):
        ch.step()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record(st); ch.step(); b.record(st)
    torch.cuda.synchronize()
    d = ch.gemm_variant
    ch.close()
    return statistics.median(a.elapsed_time(b) for a, b in ev), d


cases = [(7, 1), (7, 2), (7, 4), (7, 8), (8, 1), (8, 2), (8, 4), (8, 8), (9, 8), (9, 4)]
if len(sys.argv) > 1:
    cases = [tuple(int(x) for x in a.split(":")) for a in sys.argv[1:]]
for m, parts in cases:
    N = rd.count_words(m)
    r0, r1 = D.panel_bounds(N, parts, 0)
    plan = rd.rd_dense_step_plan(r1 - r0, N)
    res = {}
    for mode in (1, 2, 1, 2):
        rd.rd_set_gemm_tma(mode)
        t, d = med(m, r0, r1, reps=10 if m < 9 else 3)
        res.setdefault(mode, []).append((t, d))
    rd.rd_set_gemm_tma(1)
    terms = (r1 - r0) * N * N
    print(f"m={m} p={parts} rows=[{r0},{r1}) plan t{plan[0]}/{'tail' if plan[2] else 's'}{plan[1]} " +
          "  ".join(f"tma{k} " + " ".join(f"{t:.4f} ms (d={d}, {terms / t / 1e9:.1f} T)" for t, d in v)
                    for k, v in res.items()), flush=True)
