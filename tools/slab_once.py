"""A few m-order structured steps in slab mode (profiling target)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2409_17658_b200 as rd  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 9
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
ch = rd.Chain(m, alpha_max=10, method=1, stream=torch.cuda.current_stream())
for _ in range(steps):
    ch.step()
torch.cuda.synchronize()
ch.close()
print("ok")
