"""NEXT-2 beyond one GPU's ring: Algorithm 2 for m = 11 (N = 191476) on ONE B200 with the
panel-sequential structured driver (dist.power_sequence_panels).  Writes a JSON record."""
import json
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2409_17658_b200 as rd  # noqa: E402
from paper_2409_17658_b200 import dist as D  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 11
kmax = int(sys.argv[2]) if len(sys.argv) > 2 else 45
rows = int(sys.argv[3]) if len(sys.argv) > 3 else 57344
out = sys.argv[4] if len(sys.argv) > 4 else "gpurun_out/m11_chain.json"
t0 = time.time()
res = D.power_sequence_panels(m, kmax, alpha_max=5, panel_rows=rows, method=1,
                              progress=lambda p: print(json.dumps(p), flush=True))
res["total_s"] = round(time.time() - t0, 1)
res["m"], res["N"], res["kmax"] = m, rd.count_words(m), kmax
res["gpu"] = torch.cuda.get_device_name(0)
print(json.dumps({k: res[k] for k in ("m", "N", "found", "n0", "alpha", "beta", "k_stop", "total_s")}), flush=True)
print(json.dumps(res["diag"][:res["k_stop"] + 1]), flush=True)
with open(out, "w") as f:
    json.dump(res, f, indent=1)
