"""One profiled m = 7 dense step under a forced split form, for ncu (DESIGN.md §5 "Wave
quantisation"): python tools/m7_profile.py <plain|s4|tail2|tail5|t64s2|skfull|skhyb> [m] — 4 warm steps,
then the same step again (profile the 5th GEMM launch)."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2409_17658_b200 as rd  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "plain"
m = int(sys.argv[2]) if len(sys.argv) > 2 else 7
tn, n, tail = {"plain": (128, 1, 0), "s4": (128, 4, 0), "tail2": (128, 2, 2), "tail5": (128, 5, 2),
               "t64s2": (64, 2, 0), "skfull": (128, 1, 0), "skhyb": (128, 1, 0)}[cfg]
rd.rd_set_stream_k({"skfull": 3, "skhyb": 2}.get(cfg, 0))
rd.rd_set_gemm_tma(0)
rd.rd_set_gemm_tile(tn)
rd.rd_set_split_tail(tail)
rd.rd_set_split_k(n if n > 1 else 0)
ch = rd.Chain(m, alpha_max=10, stream=torch.cuda.current_stream())
for _ in range(5):
    ch.step()
torch.cuda.synchronize()
ch.close()
