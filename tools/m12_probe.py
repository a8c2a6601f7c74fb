"""m = 12 feasibility probe: one structured row panel (build time, memory, step times)."""
import json
import resource
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2409_17658_b200 as rd  # noqa: E402

m, rows, steps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
t0 = time.time()
ch = rd.Chain(m, alpha_max=5, row_begin=0, row_end=rows, method=1)
torch.cuda.synchronize()
tb = time.time() - t0
free, total = torch.cuda.mem_get_info()
rec = {"m": m, "N": ch.N, "rows": rows, "build_s": round(tb, 2), "dev_free_gb": round(free / 1e9, 1),
       "dev_total_gb": round(total / 1e9, 1), "host_maxrss_gb": round(resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6, 2),
       "terms_per_step": ch.terms_per_step}
print(json.dumps(rec), flush=True)
for k in range(2, 2 + steps):
    ts = time.time()
    s = ch.step().cpu().numpy()
    print(json.dumps({"k": k, "step_s": round(time.time() - ts, 3), "diag": int(s[0])}), flush=True)
ch.close()
