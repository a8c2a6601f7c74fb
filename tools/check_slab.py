"""Structured step: slab mode (2) vs byte (1) vs 16-bit (0) — identical powers, diag and
per-alpha decisions — and per-mode step time (CUDA events)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2409_17658_b200 as rd  # noqa: E402

ms = [int(x) for x in sys.argv[1:]] or [5, 7, 8, 9]
for m in ms:
    res = {}
    for mode in (2, 1, 0):
        rd.rd_set_sparse_bytes(mode)
        ch = rd.Chain(m, alpha_max=10, method=1, stream=torch.cuda.current_stream())
        st = []
        K = 30 if m <= 8 else 28
        for k in range(2, K + 1):
            s = ch.step().cpu().numpy()
            st.append(s)
        rows = ch.read_rows(K)
        dec = [[rd.rd_stats_decide(s, 10, k + 2, only_alpha=a) for a in range(1, min(10, k + 1) + 1)]
               for k, s in enumerate(st)]
        diag = [int(s[0]) for s in st]
        # timing
        reps = 20 if m <= 8 else 6
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            ch.step()
        e1.record()
        torch.cuda.synchronize()
        dt = e0.elapsed_time(e1) / reps
        res[mode] = (rows, dec, diag)
        print(f"m={m} mode={mode} step={dt:.3f} ms  {ch.terms_per_step / dt / 1e9:.3f} T terms/s", flush=True)
        ch.close()
    for mode in (1, 0):
        assert (res[mode][0] == res[2][0]).all(), (m, mode, "rows")
        assert res[mode][2] == res[2][2], (m, mode, "diag")
        assert res[mode][1] == res[2][1], (m, mode, "decisions")
    print(f"m={m}: modes 2/1/0 identical (rows of A^K, diag, decisions)", flush=True)
rd.rd_set_sparse_bytes(2)
