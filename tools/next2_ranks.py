"""NEXT-2 across ranks: m = 10 dense and structured through
the row-panel driver (dist.power_sequence, packed operand broadcast) and m = 11 structured
through the panel-sequential driver over ranks (dist.power_sequence_panels with a group),
run as WORLD_SIZE ranks.  On a single-GPU box the ranks share cuda:0 and reduce over gloo
(RD_DIST_BACKEND=gloo RD_FORCE_DEVICE=0): a functional multi-rank run, not a scaling number.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/next2_ranks.py OUT.json
"""
import json
import os
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2409_17658_b200 as rd  # noqa: E402
from paper_2409_17658_b200 import dist as D  # noqa: E402

out_path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/next2_ranks.json"
which = sys.argv[2].split(",") if len(sys.argv) > 2 else ["10d", "10s", "11s"]
dev = int(os.environ.get("RD_FORCE_DEVICE", os.environ.get("LOCAL_RANK", "0")))
torch.cuda.set_device(dev)
backend = os.environ.get("RD_DIST_BACKEND", "nccl")
dist.init_process_group(backend) if backend != "nccl" else dist.init_process_group(
    "nccl", device_id=torch.device("cuda", dev))
world, rank = dist.get_world_size(), dist.get_rank()
rec = {"world": world, "backend": backend, "gpu": torch.cuda.get_device_name(dev),
       "devices": torch.cuda.device_count(), "runs": {}}


def keep(name, res, t):
    k = res["k_stop"]
    rec["runs"][name] = {"found": res["found"], "triple": [res["n0"], res["alpha"], res["beta"]], "k_stop": k,
                         "gamma_3_to_kstop": res["diag"][3:k + 1], "seconds": round(t, 2),
                         **({"t_build": round(res["t_build"], 3), "t_chain": round(res["t_chain"], 3)}
                            if "t_build" in res else {})}
    if rank == 0:
        print(json.dumps({name: rec["runs"][name]}), flush=True)


for w in which:
    dist.barrier()
    t0 = time.time()
    if w == "10d":     # dense GEMM chain, row panels, A's packed operand broadcast from rank 0
        res = D.power_sequence(10, 50, 10, broadcast=True)
    elif w == "10s":   # structured chain, row panels
        res = D.power_sequence(10, 50, 10, method=1)
    elif w == "11s":   # structured, panel-sequential over ranks (ring of 6 powers per panel)
        res = D.power_sequence_panels(11, 45, alpha_max=5, panel_rows=24576, method=1)
    else:
        continue
    torch.cuda.synchronize()
    keep(w, res, time.time() - t0)
if rank == 0:
    with open(out_path, "w") as f:
        json.dump(rec, f, indent=1)
dist.destroy_process_group()
