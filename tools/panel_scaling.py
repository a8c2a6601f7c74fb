"""One rank's share of a power step at p ranks: the step time of the largest row panel of the
p-way split (dist.panel_bounds), on one GPU, CUDA events.  Implied compute-side strong-scaling
efficiency T_1 / (p * T_p) (the per-step all_reduce of 164 B and host sync come on top)."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2409_17658_b200 as rd  # noqa: E402
from paper_2409_17658_b200 import dist as D  # noqa: E402

out = {}
# arguments: orders, "10s" = the structured step only
for arg in sys.argv[1:] or ["8", "9"]:
    m, methods = (int(arg[:-1]), (1,)) if arg.endswith("s") else (int(arg), (0, 1))
    N = rd.count_words(m)
    t1 = None
    for p in (1, 2, 4, 8):
        # the slowest rank holds the largest panel
        r0, r1 = max((D.panel_bounds(N, p, r) for r in range(p)), key=lambda b: b[1] - b[0])
        for method in methods:
            ch = rd.Chain(m, alpha_max=10, row_begin=r0, row_end=r1, method=method)
            for _ in range(3):
                ch.step()
            reps = 3 if (m == 9 and method == 0 and p <= 2) else 10
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                ch.step()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            ch.close()
            key = f"m{m}_{'dense' if method == 0 else 'structured'}"
            out.setdefault(key, {})[p] = {"rows": r1 - r0, "ms": round(ms, 3)}
    for key, d in out.items():
        if not key.startswith(f"m{m}_"):
            continue
        for p, v in d.items():
            v["eff"] = round(d[1]["ms"] / (p * v["ms"]), 3)
print(json.dumps(out, indent=1))
