"""One warm dense Algorithm 2 at order m through the device-resident small-order kernel, for ncu
(profile the second small_chain_kernel launch): python tools/small_profile.py [m]"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2409_17658_b200 as rd  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 3
torch.cuda.init()
for _ in range(2):
    r = rd.rd_power_sequence(m, 50, 10)
print(r["n0"], r["alpha"], r["beta"], r["k_stop"])
