"""Dense step time per order with the split-K rule on and off (median of 10, CUDA events),
also for row panels (the per-rank share at 8 ranks)."""
import statistics
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2409_17658_b200 as rd  # noqa: E402
from paper_2409_17658_b200 import dist as D  # noqa: E402


def med(m, r0, r1, reps=10):
    st = torch.cuda.current_stream()
    ch = rd.Chain(m, alpha_max=10, row_begin=r0, row_end=r1, stream=st)
    for _ in range(4):
        ch.step()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record(st); ch.step(); b.record(st)
    torch.cuda.synchronize()
    ch.close()
    return statistics.median(a.elapsed_time(b) for a, b in ev)


for m, parts in ((6, 1), (7, 1), (8, 1), (8, 8), (9, 8)):
    N = rd.count_words(m)
    r0, r1 = D.panel_bounds(N, parts, 0)
    out = []
    for on in (True, False):
        rd.rd_set_split_k(on)
        out.append(med(m, r0, r1))
    rd.rd_set_split_k(True)
    print(f"m={m} rows=[{r0},{r1}) split-rule {out[0]:.3f} ms  no-split {out[1]:.3f} ms", flush=True)
