"""DPX column count (rd_set_gemm_variant) under the TMA mainloop: identical powers and stats,
and the median chain-step time (CUDA events), at m = 8 and m = 9."""
import statistics
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2409_17658_b200 as rd  # noqa: E402


def run(m, d, steps=6, reps=5):
    rd.rd_set_gemm_variant(d)
    st = torch.cuda.current_stream()
    ch = rd.Chain(m, alpha_max=10, stream=st)
    stats = [ch.step().cpu().numpy().copy() for _ in range(steps)]
    rows = ch.read_rows(ch.k)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record(st); ch.step(); b.record(st)
    torch.cuda.synchronize()
    ch.close()
    rd.rd_set_gemm_variant(-1)
    return np.stack(stats), rows, statistics.median(a.elapsed_time(b) for a, b in ev)


for m in (8, 9):
    base = None
    for d in ((3, 13, 4, 14, 3) if len(sys.argv) < 2 else [int(x) for x in sys.argv[1:]]):
        s, x, t = run(m, d)
        if base is None:
            base = (s, x)
        same = bool((s == base[0]).all() and (x == base[1]).all())
        print(f"m={m} dpx_cols={d} identical={same} step {t:.3f} ms", flush=True)
