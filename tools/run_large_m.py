"""Algorithm 2 for a large m on one GPU with per-step progress (NEXT-2: m = 10).

Prints one JSON line per power (k, diag, stats decision, step seconds) and a final line
with (n0, alpha, beta), every gamma(n) = diag[n] and the timings.  The diag values are
pinned in tests by Cor 12 (5 | n) and the row DP for small n (tests/test_gpu_large_m.py).
"""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2409_17658_b200 as rd  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 10
kmax = int(sys.argv[2]) if len(sys.argv) > 2 else 50
am = int(sys.argv[3]) if len(sys.argv) > 3 else 10
out = sys.argv[4] if len(sys.argv) > 4 else None

t0 = time.time()
ch = rd.Chain(m, alpha_max=am)
torch.cuda.synchronize()
tb = time.time() - t0
N = ch.N
diag = {1: ch.diag1}
found = None
rows = []
for k in range(2, kmax + 1):
    ts = time.time()
    s = ch.step().cpu().numpy()
    dt = time.time() - ts
    diag[k] = int(s[0])
    dec = rd.rd_stats_decide(s, am, k)
    rec = {"k": k, "diag": diag[k], "decision": dec, "step_s": round(dt, 3),
           "gops": round(float(N) ** 3 / dt / 1e9, 1)}
    rows.append(rec)
    print(json.dumps(rec), flush=True)
    if dec:
        found = (k - dec[0], dec[0], dec[1])
        break
total = time.time() - t0
res = {"m": m, "N": N, "triple": found, "k_stop": k, "diag": diag, "build_s": round(tb, 2),
       "chain_s": round(total - tb, 2), "total_s": round(total, 2),
       "gpu": torch.cuda.get_device_name(0)}
print(json.dumps(res), flush=True)
if out:
    with open(out, "w") as f:
        json.dump({"result": res, "steps": rows}, f, indent=1)
