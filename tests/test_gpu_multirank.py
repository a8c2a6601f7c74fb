"""The multi-rank drivers on one GPU: 2 processes on cuda:0 with gloo (host-side) collectives.

No kernel waits on another rank (the ranks only meet in the host collectives), so this runs
the real row-panel, broadcast and all-gather drivers end to end on the single GPU the test
box has; results must equal the oracle.  (NCCL needs distinct devices; bench.py uses NCCL.)"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


WORKER = r'''
import json, os, sys
sys.path.insert(0, os.environ["ROOT"])
import torch, torch.distributed as dist
import paper_2409_17658_b200 as rd
from paper_2409_17658_b200 import dist as D
torch.cuda.set_device(0)
dist.init_process_group("gloo")
out = {}
for m in (5, 6):
    r = D.power_sequence(m, 50, 10)
    out["rep%d" % m] = [r["n0"], r["alpha"], r["beta"], r["k_stop"], r["diag"][1:r["k_stop"] + 1]]
    r = D.power_sequence(m, 50, 10, broadcast=True)
    out["bc%d" % m] = [r["n0"], r["alpha"], r["beta"], r["k_stop"], r["diag"][1:r["k_stop"] + 1]]
    r = D.power_sequence(m, 50, 10, method=1)
    out["st%d" % m] = [r["n0"], r["alpha"], r["beta"], r["k_stop"], r["diag"][1:r["k_stop"] + 1]]
r = D.power_sequence_allgather(5, 50, 10)
out["ag5"] = [r["n0"], r["alpha"], r["beta"], r["k_stop"], r["diag"][1:r["k_stop"] + 1]]
torch.cuda.synchronize()
if dist.get_rank() == 0:
    print("RESULT " + json.dumps(out), flush=True)
dist.destroy_process_group()
'''


def test_two_ranks_one_gpu_gloo_drivers(tmp_path):
    script = tmp_path / "w.py"
    script.write_text(WORKER)
    env = dict(os.environ, ROOT=ROOT, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()), WORLD_SIZE="2")
    procs = [subprocess.Popen([sys.executable, str(script)], env=dict(env, RANK=str(r), LOCAL_RANK=str(r)),
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True) for r in range(2)]
    outs = [p.communicate(timeout=600)[0] for p in procs]
    assert all(p.returncode == 0 for p in procs), outs
    line = [l for l in outs[0].splitlines() if l.startswith("RESULT ")][0]
    res = json.loads(line[7:])
    for m in (5, 6):
        ref = O.power_chain(m, 50, 10, 0)
        want = [ref["n0"], ref["alpha"], ref["beta"], ref["k_stop"], ref["diag"][1:ref["k_stop"] + 1]]
        assert res["rep%d" % m] == want
        assert res["bc%d" % m] == want
        assert res["st%d" % m] == want
    ref = O.power_chain(5, 50, 10, 0)
    assert res["ag5"] == [ref["n0"], ref["alpha"], ref["beta"], ref["k_stop"], ref["diag"][1:ref["k_stop"] + 1]]


def test_bench_two_ranks_one_gpu_gloo():
    # bench.py under torchrun with 2 ranks (gloo, one GPU): the line is well formed and the
    # detected triple is right; not a performance number
    env = dict(os.environ, RD_DIST_BACKEND="gloo", RD_FORCE_DEVICE="0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--order-m", "7", "--steps", "3", "--warmup", "22", "--no-cpu-baseline", "--ttp-m", "5"]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["backend"] == "gloo"
    assert d["config"]["detected"] == [21, 5, 16]
    assert d["e2e"]["triple"] == [21, 5, 16]
    assert d["time_to_periodicity"]["5"]["triple"] == [16, 5, 12]


def test_bench_self_launch_two_ranks():
    # `bench.py --gpus 2` WITHOUT torchrun (the driver's plain invocation): bench.py starts the
    # two ranks itself; the gloo hook puts both on cuda:0 (functional check, not a perf number)
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    env.update(RD_DIST_BACKEND="gloo", RD_FORCE_DEVICE="0")
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--order-m", "7", "--steps", "3",
           "--warmup", "22", "--no-cpu-baseline", "--ttp-m", "5", "--ttp-structured-only-m", "--gops-m",
           "--invariance-m", "0"]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["backend"] == "gloo"
    assert d["config"]["detected"] == [21, 5, 16]
    assert d["e2e"]["triple"] == [21, 5, 16]
    assert d["time_to_periodicity"]["5"]["triple"] == [16, 5, 12]


PEER_WORKER = r'''
import json, os, sys
sys.path.insert(0, os.environ["ROOT"])
import numpy as np
import torch, torch.distributed as dist
import paper_2409_17658_b200 as rd
from paper_2409_17658_b200 import dist as D
torch.cuda.set_device(0)
dist.init_process_group("gloo")
out = {}
for m in (5, 6, 7):
    r = D.power_sequence_peer(m, 50, 10)
    out["peer%d" % m] = [r["n0"], r["alpha"], r["beta"], r["k_stop"], r["diag"][1:r["k_stop"] + 1]]
# rows of A^6 at m = 6 from the peer chain, gathered on rank 0 (checked against the oracle)
ch = D.peer_chain(6, 4)
dist.barrier()
for k in range(2, 7):
    s = ch.step()
    dist.all_reduce(s, op=dist.ReduceOp.MIN)
    s.cpu()
rows = ch.read_rows(6)
got = [None] * dist.get_world_size()
dist.all_gather_object(got, rows.tolist())
dist.barrier()
ch.close()
if dist.get_rank() == 0:
    out["rows6"] = [r for part in got for r in part]
    print("RESULT " + json.dumps(out), flush=True)
dist.destroy_process_group()
'''


def test_two_ranks_one_gpu_peer_allgather(tmp_path):
    # the fused peer all-gather form across 2 processes: each GEMM reads the other process's
    # ring through a CUDA IPC mapping (the NVLink path on a multi-GPU node)
    script = tmp_path / "p.py"
    script.write_text(PEER_WORKER)
    env = dict(os.environ, ROOT=ROOT, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()), WORLD_SIZE="2")
    procs = [subprocess.Popen([sys.executable, str(script)], env=dict(env, RANK=str(r), LOCAL_RANK=str(r)),
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True) for r in range(2)]
    outs = [p.communicate(timeout=600)[0] for p in procs]
    assert all(p.returncode == 0 for p in procs), outs
    line = [l for l in outs[0].splitlines() if l.startswith("RESULT ")][0]
    res = json.loads(line[7:])
    for m in (5, 6, 7):
        ref = O.power_chain(m, 50, 10, 0)
        assert res["peer%d" % m] == [ref["n0"], ref["alpha"], ref["beta"], ref["k_stop"],
                                     ref["diag"][1:ref["k_stop"] + 1]], m
    A = O.matrix(6)
    P = A.copy()
    for _ in range(5):
        P = O.minplus(P, A, skip=True)
    want = np.where(P >= O.INF, 0x3FFF, P).astype(np.int16)
    assert (np.array(res["rows6"], dtype=np.int16) == want).all()


def test_bench_two_ranks_one_gpu_gloo_peer_form():
    # bench.py --form peer under torchrun with 2 ranks on one GPU (gloo): each rank's GEMM
    # reads the other's ring through CUDA IPC; the detected triple is right (not a perf number)
    env = dict(os.environ, RD_DIST_BACKEND="gloo", RD_FORCE_DEVICE="0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--order-m", "7", "--form", "peer", "--steps", "3", "--warmup", "22",
           "--no-cpu-baseline", "--no-e2e"]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["form"] == "peer"
    assert d["config"]["detected"] == [21, 5, 16]
    assert d["gpu_launches"] == 2 * 3 * 2
