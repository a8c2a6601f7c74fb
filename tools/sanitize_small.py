"""Small workload touching every librd kernel with ragged sizes (for compute-sanitizer)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2409_17658_b200 as rd  # noqa: E402
from rd_inputs import operand  # noqa: E402

torch.cuda.set_device(0)
for N in (1, 33, 130, 300):
    A = torch.from_numpy(operand(N, N, 1, inf_frac=0.1)).cuda()
    B = torch.from_numpy(operand(N, N, 2, inf_frac=0.1)).cuda()
    C = rd.rd_minplus_mul(A, B)
    rd.rd_minplus_mul_acc(A, N, B, N, C, N, N, N, N)
for v in (0, 2, 3, 4, 8):
    rd.rd_set_gemm_variant(v)
    rd.rd_minplus_mul(torch.from_numpy(operand(257, 257, 3)).cuda(), torch.from_numpy(operand(257, 257, 4)).cuda())
rd.rd_set_gemm_variant(-1)
for method in (0, 1):
    for m in (3, 5):
        print(m, method, rd.rd_power_sequence(m, 50, method=method)["n0"])
    ch = rd.Chain(5, alpha_max=4, row_begin=100, row_end=287, method=method)
    for _ in range(6):
        ch.step()
    ch.read_rows(7)
    ch.close()
print(rd.rd_power_sequence_matrix(rd.rd_build_matrix_border(), 40, 5, 0, 1)["n0"])
X = torch.from_numpy(operand(90, 77, 5, inf_frac=0.2)).cuda()
P = [torch.from_numpy(operand(90, 77, 6 + a, inf_frac=0.2)).cuda() for a in range(3)]
s = torch.empty(rd.rd_stats_len(10), dtype=torch.int32, device="cuda")
rd.rd_panel_stats(X, P, 5, 10, s)
torch.cuda.synchronize()
print("sanitize workload done")
