"""Times rd_minplus_mul_ex / _acc and the chain step at one order (CUDA events)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2409_17658_b200 as rd  # noqa: E402
from rd_inputs import operand, power_like, sparse_like  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 21909
m = {21909: 9, 7411: 8, 2507: 7}.get(N, 9)


def t(fn, reps=3):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


X = torch.from_numpy(power_like(N, N, m, seed=1)).cuda()
S = torch.from_numpy(sparse_like(N, m, seed=2)).cuda()
C = torch.empty((N, N), dtype=torch.int16, device="cuda")
for name, A, B in (("dense x sparse", X, S), ("sparse x dense", S, X), ("dense x dense", X, X)):
    ms = t(lambda: rd.rd_minplus_mul_ex(A, N, B, N, C, N, N, N, N))
    print(f"mul_ex {name:15s} N={N}: {ms:.2f} ms  {N**3/ms/1e9:.1f} Gop/s", flush=True)
    ms = t(lambda: rd.rd_minplus_mul_acc(A, N, B, N, C, N, N, N, N))
    print(f"mul_acc {name:14s} N={N}: {ms:.2f} ms  {N**3/ms/1e9:.1f} Gop/s", flush=True)
ch = rd.Chain(m, alpha_max=10)
for _ in range(3):
    ch.step()
ms = t(lambda: ch.step())
print(f"chain step m={m}: {ms:.2f} ms  {N**3/ms/1e9:.1f} Gop/s")
