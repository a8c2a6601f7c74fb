"""Dense chain step time (median of 10, CUDA events) per order / row panel under forced tile
widths (128, 64), split-K counts (1..4, every tile split; in-kernel fixup) and tail splits
(2..6: the whole waves unsplit, the last partial wave's tiles split), plus the library's
default choice: the data behind the wave model of rd_chain_step (DESIGN.md §5 "Wave
quantisation")."""
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


cases = [(6, 1), (7, 1), (7, 2), (7, 4), (8, 1), (8, 2), (8, 4), (8, 8), (9, 8)]
if len(sys.argv) > 1:
    cases = [tuple(int(x) for x in a.split(":")) for a in sys.argv[1:]]
for m, parts in cases:
    N = rd.count_words(m)
    r0, r1 = D.panel_bounds(N, parts, 0)
    terms = (r1 - r0) * N * N
    res = {}
    for tn in (128, 64):
        rd.rd_set_gemm_tile(tn)
        rd.rd_set_gemm_tma(1)   # the library's policy: TMA for 128-wide steps of >= 64 stages
        rd.rd_set_split_tail(0)
        for n in (1, 2, 3, 4):
            rd.rd_set_split_k(0 if n == 1 else n)
            res[f"t{tn}/s{n}"] = med(m, r0, r1, reps=10 if m < 9 else 3)
        rd.rd_set_split_tail(2)
        for n in (2, 3, 4, 5, 6):
            rd.rd_set_split_k(n)
            if rd.rd_dense_step_plan(r1 - r0, N)[2]:   # a tail exists
                res[f"t{tn}/tail{n}"] = med(m, r0, r1, reps=10 if m < 9 else 3)
    rd.rd_set_gemm_tile(0)
    rd.rd_set_gemm_tma(1)
    rd.rd_set_split_k(1)
    rd.rd_set_split_tail(1)
    res["default"] = med(m, r0, r1, reps=10 if m < 9 else 3)
    best = min(res, key=res.get)
    print(f"m={m} p={parts} rows=[{r0},{r1}) best {best} " +
          "  ".join(f"{k} {v:.4f} ms ({terms / v / 1e9:.1f} T)" for k, v in res.items()), flush=True)
