"""Median time of the int32 product rd_minplus_mul32 at N = 7411 (uniform [0, 2^29), 1 % inf;
the bench's operand_invariance.mul32 case) for the librd build named by RD_LIB (A/B)."""
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2409_17658_b200 as rd  # noqa: E402
from rd_inputs import operand  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 7411
A = torch.from_numpy(operand(N, N, 7, inf_frac=0.01, hi=2**29 - 1, inf=rd.RD_INF32, dtype=np.int32)).cuda()
B = torch.from_numpy(operand(N, N, 8, inf_frac=0.01, hi=2**29 - 1, inf=rd.RD_INF32, dtype=np.int32)).cuda()
for _ in range(2):
    rd.rd_minplus_mul32(A, B)
torch.cuda.synchronize()
ts = []
for _ in range(7):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); rd.rd_minplus_mul32(A, B); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
t = statistics.median(ts)
print(f"{os.path.basename(os.environ.get('RD_LIB', 'librd.so'))} mul32 N={N}: {t:.3f} ms {float(N) ** 3 / t / 1e9:.1f} Gop/s", flush=True)
