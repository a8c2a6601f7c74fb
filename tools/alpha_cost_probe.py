"""Cost of the fused periodicity stats in the dense step: median step time (CUDA events) with
alpha_max = 1, 5, 10 at m = 7, 8 and 10 at m = 9 (the epilogue reads alpha_max earlier tiles).
RD_LIB=<path> runs another build of librd.so (A/B)."""
import statistics
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2409_17658_b200 as rd  # noqa: E402

st = torch.cuda.current_stream()
for m in (7, 8, 9):
    for am in ((1, 5, 10) if m < 9 else (10,)):
        ch = rd.Chain(m, alpha_max=am, stream=st)
        for _ in range(am + 2):
            ch.step()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10 if m < 9 else 3)]
        for a, b in ev:
            a.record(st); ch.step(); b.record(st)
        torch.cuda.synchronize()
        ch.close()
        print(f"m={m} alpha_max={am}: {statistics.median(a.elapsed_time(b) for a, b in ev):.4f} ms", flush=True)
