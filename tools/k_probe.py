"""Per-term rate of the generic product vs K at fixed M = N (per-CTA fixed costs show up as a
lower rate at small K)."""
import statistics
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2409_17658_b200 as rd  # noqa: E402

st = torch.cuda.current_stream()
M = N = 9472   # 74 x 74 tiles = 5476 CTAs = 18.5 waves
for K in (4096, 9472, 18944, 37888, 75776):
    X = torch.randint(0, 200, (M, K), dtype=torch.int16, device="cuda")
    Y = torch.randint(0, 200, (K, N), dtype=torch.int16, device="cuda")
    C = torch.empty((M, N), dtype=torch.int16, device="cuda")
    f = lambda: rd.rd_minplus_mul_ex(X, K, Y, N, C, N, M, N, K)
    f()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(5)]
    for a, b in ev:
        a.record(st); f(); b.record(st)
    torch.cuda.synchronize()
    ms = statistics.median(a.elapsed_time(b) for a, b in ev)
    print(f"K={K}: {ms:.3f} ms  {M * N * K / ms / 1e9:.1f} T op/s", flush=True)
    del X, Y, C
