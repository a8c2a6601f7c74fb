"""Multi-rank row-panel driver on CPU: world_size 2 (and 3) over gloo.

The partition, the MIN-reduction of the stats vector and the shared decision loop of
paper_2409_17658_b200.dist.power_sequence run unchanged; only the per-panel product is
replaced by an oracle-backed panel (test code) since there is no GPU here.  The result
must equal the oracle's single-process chain (and Table 2).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2409_17658_b200 import dist as rdist

OINF = int(O.INF)
RINF = 0x3FFF


class OraclePanel:
    """Rows [r0, r1) of A^k by the oracle, with the stats vector in the library's
    MIN-reducible layout (rd.h rd_chain_step)."""

    def __init__(self, m, alpha_max, r0, r1):
        self.A = O.matrix(m)
        self.r0, self.r1, self.am = r0, r1, alpha_max
        self.k = 1
        self.ring = {1: self.A[r0:r1].copy()}

    def step(self):
        k = self.k + 1
        X = O.minplus(self.ring[self.k], self.A, skip=True)
        self.ring[k] = X
        s = rdist.neutral_stats(self.am)
        n = X.shape[0]
        d = [X[i, self.r0 + i] for i in range(n)]
        s[0] = min(min(d), RINF) if d else 2**31 - 1
        for a in range(1, min(self.am, k - 1) + 1):
            P = self.ring[k - a]
            fx, fp = X != OINF, P != OINF
            both = fx & fp
            diff = X[both].astype(np.int64) - P[both].astype(np.int64)
            e = 1 + 4 * (a - 1)
            if diff.size:
                s[e], s[e + 1] = int(diff.min()), -int(diff.max())
            s[e + 2] = -1 if (fx != fp).any() else 0
            s[e + 3] = -1 if both.any() else 0
        self.ring.pop(k - self.am - 1, None)
        self.k = k
        return torch.from_numpy(s)

    @property
    def diag1(self):
        d = [int(self.A[i, i]) for i in range(self.r0, self.r1) if self.A[i, i] != OINF]
        return min(d) if d else 2**31 - 1

    def close(self):
        pass


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, m, policy, alpha_max, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A = O.matrix(m)
        d = np.diag(A)
        res = rdist.power_sequence(m, 50, alpha_max, policy,
                                   chain_factory=lambda m_, am_, a, b: OraclePanel(m_, am_, a, b),
                                   diag1=int(d[d != OINF].min()))
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def _run(world, m, policy=0, alpha_max=10):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, m, policy, alpha_max, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


def test_panel_bounds_cover_and_balance():
    for N in (1, 33, 127, 128, 129, 2507, 21909):
        for W in (1, 2, 3, 4, 8):
            b = [rdist.panel_bounds(N, W, r) for r in range(W)]
            assert b[0][0] == 0 and b[-1][1] == N
            for (a0, a1), (c0, c1) in zip(b, b[1:]):
                assert a1 == c0
            tiles = [(e - s + 127) // 128 for s, e in b]
            assert max(tiles) - min(tiles) <= 1
            assert all(s % 128 == 0 for s, e in b if e > s)


def test_neutral_stats_is_min_identity():
    s = rdist.neutral_stats(3)
    x = np.array([7, 2, -2, -1, -1] + [5, -5, 0, -1] * 2, dtype=np.int32)
    assert (np.minimum(s, x) == x).all()


@pytest.mark.parametrize("m", [3, 5])
def test_gloo_world2_equals_single_process(m):
    out = _run(2, m)
    ref = O.power_chain(m, 50, 10, 0)
    for r in (0, 1):
        res = out[r]
        assert (res["n0"], res["alpha"], res["beta"], res["k_stop"]) == (ref["n0"], ref["alpha"], ref["beta"],
                                                                         ref["k_stop"])
        assert res["diag"][1:res["k_stop"] + 1] == ref["diag"][1:ref["k_stop"] + 1]


def test_gloo_world3_paper_compat_table2(golden):
    # m = 4: 97 rows -> one 128-row tile -> ranks 1 and 2 hold empty panels
    out = _run(3, 4, policy=1, alpha_max=5)
    want = tuple(golden("table2_periods.json")["table2"]["4"])
    for r in range(3):
        assert (out[r]["n0"], out[r]["alpha"], out[r]["beta"]) == want


# ------------------------------------------------------------ all-gather form --
def _acc_oracle(A_rows, k0, k1, chunk, C):
    if k1 <= k0 or A_rows.shape[0] == 0:
        return
    a = A_rows[:, k0:k1].numpy().astype(np.int32)
    b = chunk.numpy().astype(np.int32)
    a[a >= RINF] = OINF
    b[b >= RINF] = OINF
    P = O.minplus(a, b)
    P[P == OINF] = RINF
    C.copy_(torch.from_numpy(np.minimum(C.numpy(), P.astype(np.int16))))


def _stats_oracle(r0, am):
    def f(cur, prevs):
        X = cur.numpy().astype(np.int64)
        s = rdist.neutral_stats(am)
        d = [X[i, r0 + i] for i in range(X.shape[0])]
        s[0] = min(d) if d else 2**31 - 1
        for a, P in enumerate(prevs, start=1):
            P = P.numpy().astype(np.int64)
            fx, fp = X < RINF, P < RINF
            both = fx & fp
            e = 1 + 4 * (a - 1)
            if both.any():
                diff = X[both] - P[both]
                s[e], s[e + 1] = int(diff.min()), -int(diff.max())
            s[e + 2] = -1 if (fx != fp).any() else 0
            s[e + 3] = -1 if both.any() else 0
        return torch.from_numpy(s)
    return f


def _ag_worker(rank, world, port, m, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A = O.matrix(m)
        A16 = np.where(A == OINF, RINF, A).astype(np.int16)
        N = A.shape[0]
        r0, _ = rdist.panel_bounds(N, world, rank)
        # generic product first: C = X (x) A with X, A row/k-sharded
        rng = np.random.default_rng(3)
        X = rng.integers(0, 50, size=(N, N)).astype(np.int16)
        bounds = [rdist.panel_bounds(N, world, s) for s in range(world)]
        a, b = bounds[rank]
        C = rdist.minplus_mul_allgather(torch.from_numpy(X[a:b].copy()), torch.from_numpy(A16[a:b].copy()),
                                        bounds, acc=_acc_oracle)
        res = rdist.power_sequence_allgather(m, 50, 10, 0, acc=_acc_oracle, stats=_stats_oracle(r0, 10), A=A16)
        q.put((rank, (res, (a, b), C.numpy())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,m", [(2, 5), (3, 5)])
def test_gloo_allgather_product_and_chain(world, m):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_ag_worker, args=(r, world, port, m, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    A = O.matrix(m)
    N = A.shape[0]
    rng = np.random.default_rng(3)
    X = rng.integers(0, 50, size=(N, N)).astype(np.int32)
    want = O.minplus(X, A)
    want[want == OINF] = RINF
    ref = O.power_chain(m, 50, 10, 0)
    for r in range(world):
        res, (a, b), C = out[r]
        assert (C == want[a:b]).all()
        assert (res["n0"], res["alpha"], res["beta"], res["k_stop"]) == (ref["n0"], ref["alpha"], ref["beta"],
                                                                         ref["k_stop"])
        assert res["diag"][1:res["k_stop"] + 1] == ref["diag"][1:ref["k_stop"] + 1]


# ------------------------------------------------- peer all-gather form (fused) --
class OraclePeerPanel:
    """Stand-in for rd.AgChain on CPU: rows R_r of A^{k+1} = A (x) A^k by the oracle.  The
    GEMM's reads of the peers' ring slots are emulated by an all_gather_object of the current
    rows; the handle exchange, the stats reduction and the decision loop of
    dist.power_sequence_peer run unchanged."""

    def __init__(self, m, bounds, rank, alpha_max):
        self.A = O.matrix(m)
        self.bounds, self.rank, self.am = bounds, rank, alpha_max
        self.r0, self.r1 = bounds[rank], bounds[rank + 1]
        self.k = 1
        self.ring = {1: self.A[self.r0:self.r1].copy()}
        self.peers = {}
        d = np.diag(self.A)[self.r0:self.r1]
        self.diag1 = int(d[d != OINF].min()) if (d != OINF).any() else 2**31 - 1

    def ipc_handle(self):
        return bytes([self.rank]) * 64, (self.r1 - self.r0) * self.A.shape[0]

    def set_peer(self, s, handle=None, ring_ptr=None, slot_words=0):
        assert handle == bytes([s]) * 64
        assert slot_words == (self.bounds[s + 1] - self.bounds[s]) * self.A.shape[0]
        self.peers[s] = handle

    def step(self):
        assert len(self.peers) == len(self.bounds) - 2
        parts = [None] * (len(self.bounds) - 1)
        dist.all_gather_object(parts, self.ring[self.k])
        Ak = np.concatenate(parts, axis=0)
        k = self.k + 1
        X = O.minplus(self.A[self.r0:self.r1], Ak, skip=True)
        self.ring[k] = X
        s = rdist.neutral_stats(self.am)
        d = [X[i, self.r0 + i] for i in range(X.shape[0])]
        s[0] = min(min(d), RINF)
        for a in range(1, min(self.am, k - 1) + 1):
            P = self.ring[k - a]
            fx, fp = X != OINF, P != OINF
            both = fx & fp
            e = 1 + 4 * (a - 1)
            if both.any():
                diff = X[both].astype(np.int64) - P[both].astype(np.int64)
                s[e], s[e + 1] = int(diff.min()), -int(diff.max())
            s[e + 2] = -1 if (fx != fp).any() else 0
            s[e + 3] = -1 if both.any() else 0
        self.ring.pop(k - self.am - 1, None)
        self.k = k
        return torch.from_numpy(s)

    def close(self):
        pass


def _peer_worker(rank, world, port, m, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = rdist.power_sequence_peer(m, 50, 10, 0, factory=OraclePeerPanel)
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_peer_bounds():
    assert rdist.peer_bounds(287, 2) == [0, 256, 287]
    assert rdist.peer_bounds(21909, 8)[1:3] == [2816, 5632]
    with pytest.raises(ValueError):
        rdist.peer_bounds(287, 4)       # 3 tiles, 4 ranks: the fused form needs non-empty panels


@pytest.mark.parametrize("world,m", [(2, 5), (3, 6)])
def test_gloo_peer_allgather_chain(world, m):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_peer_worker, args=(r, world, port, m, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = O.power_chain(m, 50, 10, 0)
    for r in range(world):
        res = out[r]
        assert (res["n0"], res["alpha"], res["beta"], res["k_stop"]) == (ref["n0"], ref["alpha"], ref["beta"],
                                                                         ref["k_stop"])
        assert res["diag"][1:res["k_stop"] + 1] == ref["diag"][1:ref["k_stop"] + 1]


# --------------------------------------------- panel-sequential driver over ranks --
def _panels_worker(rank, world, port, m, panel_rows, policy, alpha_max, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = rdist.power_sequence_panels(m, 40, alpha_max, panel_rows=panel_rows, policy=policy,
                                          chain_factory=lambda m_, am_, a, b: OraclePanel(m_, am_, a, b))
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,m,rows,policy", [(2, 5, 128, 0), (3, 5, 128, 1), (2, 4, 128, 0)])
def test_gloo_panels_over_ranks_equals_single_process(world, m, rows, policy):
    """power_sequence_panels across ranks (rank r runs panels r, r + world, ...; stats arrays
    MIN-reduced; one shared decision) equals the oracle's Algorithm 2, also when a rank holds
    no panel (m = 4: one 128-row panel for 2 ranks) and under the paper-compatible policy."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    am = 5
    ps = [ctx.Process(target=_panels_worker, args=(r, world, port, m, rows, policy, am, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = O.power_chain(m, 40, am, policy)
    for r in range(world):
        res = out[r]
        assert (res["found"], res["n0"], res["alpha"], res["beta"], res["k_stop"]) == (
            ref["found"], ref["n0"], ref["alpha"], ref["beta"], ref["k_stop"]), (r, res["k_stop"])
        assert res["diag"][1:ref["k_stop"] + 1] == ref["diag"][1:ref["k_stop"] + 1]
