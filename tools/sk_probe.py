"""Dense step time (median of 10, CUDA events) per order and row panel under the wave
strategies: plain (one tile per CTA), split-K (wave model's count), 64-wide tiles, stream-K
hybrid (mode 2) and full (mode 3) with the in-kernel fixup, and the library's default plan."""
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


MODES = {"plain": (False, 0, 128), "splitk": (True, 0, 128), "t64": (False, 0, 64), "t64split": (True, 0, 64),
         "sk_hybrid": (False, 2, 128), "sk_full": (False, 3, 128), "default": (True, 0, 0)}
cases = [(6, 1), (7, 1), (7, 2), (7, 4), (8, 1), (8, 2), (8, 4), (8, 8), (9, 8)]
if len(sys.argv) > 1:
    cases = [tuple(int(x) for x in a.split(":")) for a in sys.argv[1:]]
for m, parts in cases:
    N = rd.count_words(m)
    r0, r1 = D.panel_bounds(N, parts, 0)
    res = {}
    for name, (split, sk, tn) in MODES.items():
        rd.rd_set_split_k(split)
        rd.rd_set_stream_k(sk)
        rd.rd_set_gemm_tile(tn)
        rd.rd_set_gemm_tma(0 if tn == 64 else 1)
        res[name] = med(m, r0, r1, reps=10 if m < 9 else 3)
    rd.rd_set_split_k(True)
    rd.rd_set_stream_k(0)
    rd.rd_set_gemm_tile(0)
    rd.rd_set_gemm_tma(1)
    terms = (r1 - r0) * N * N
    print(f"m={m} p={parts} rows=[{r0},{r1}) " + "  ".join(f"{k} {v:.4f} ms ({terms / v / 1e9:.1f} T)" for k, v in res.items()),
          flush=True)
