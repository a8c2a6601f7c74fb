"""Cost of the fused stats epilogue at m = 9: the chain step (GEMM + diag + 10-alpha stats,
TMA mainloop) vs the generic product of the same size (GEMM without stats, row-major output,
packing included) vs the chain step with alpha_max = 1."""
import statistics
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2409_17658_b200 as rd  # noqa: E402
from rd_inputs import operand  # noqa: E402


def timed(fn, reps=4):
    st = torch.cuda.current_stream()
    fn()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record(st); fn(); b.record(st)
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in ev)


for am in (10, 1):
    ch = rd.Chain(9, alpha_max=am)
    for _ in range(11):
        ch.step()
    print(f"chain step alpha_max={am}: {timed(ch.step):.2f} ms", flush=True)
    ch.close()
N = rd.count_words(9)
X = torch.from_numpy(operand(N, N, 1, hi=200)).cuda()
Y = torch.from_numpy(operand(N, N, 2, hi=200)).cuda()
C = torch.empty_like(X)
print(f"generic product (pack + GEMM, no stats, cp.async): {timed(lambda: rd.rd_minplus_mul_ex(X, N, Y, N, C, N, N, N, N)):.2f} ms")
