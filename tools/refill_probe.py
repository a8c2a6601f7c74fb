"""A/B of the TMA mainloop's stage refill at m = 9 (median chain-step time, CUDA events),
alternating configurations to cancel clock drift: the last warp to release a
stage refills it, mode 3) vs the default (thread 0 waits for every warp, mode 1), for dpx_cols 3 and 4."""
import statistics
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2409_17658_b200 as rd  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 9
st = torch.cuda.current_stream()
ch = rd.Chain(m, alpha_max=10, stream=st)
for _ in range(3):
    ch.step()
res = {}
for rep in range(3):
    for d in (3, 4):
        for mode, name in ((3, "last-warp"), (1, "thread0")):
            rd.rd_set_gemm_tma(mode)
            rd.rd_set_gemm_variant(d)
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(2)]
            for a, b in ev:
                a.record(st); ch.step(); b.record(st)
            torch.cuda.synchronize()
            res.setdefault(f"d={d} {name}", []).extend(a.elapsed_time(b) for a, b in ev)
rd.rd_set_gemm_tma(1)
rd.rd_set_gemm_variant(-1)
ch.close()
N = rd.count_words(m)
for k, v in res.items():
    t = statistics.median(v)
    print(f"m={m} {k}: {t:.3f} ms ({float(N) ** 3 / t / 1e9:.1f} T)  samples {['%.1f' % x for x in v]}", flush=True)
