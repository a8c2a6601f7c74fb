"""Times rd_panel_stats on m=9-sized panels (21909 x 21909 int16) against alpha_max earlier
powers (default 10; more arguments: a sweep over alpha, bytes (1 + alpha) * 2 N^2 per call)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2409_17658_b200 as rd  # noqa: E402

N = 21909
alphas = [int(a) for a in sys.argv[1:]] or [10]
g = torch.Generator(device="cuda").manual_seed(0)
cur = torch.randint(100, 140, (N, N), dtype=torch.int16, device="cuda", generator=g)
prevs = [torch.randint(40 + 2 * a, 100, (N, N), dtype=torch.int16, device="cuda", generator=g) for a in range(max(alphas))]
for am in alphas:
    s = torch.empty(rd.rd_stats_len(max(am, 1)), dtype=torch.int32, device="cuda")
    for _ in range(3):
        rd.rd_panel_stats(cur, prevs[:am], 0, max(am, 1), s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        rd.rd_panel_stats(cur, prevs[:am], 0, max(am, 1), s)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    by = (1 + am) * 2 * N * N
    print(f"panel_stats N={N} alpha={am}: {ms:.3f} ms per call (one pass), {by / ms / 1e6:.1f} GB/s algorithmic",
          flush=True)
