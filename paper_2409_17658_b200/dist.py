"""Multi-GPU power chain: one process per GPU, output row panels.

Row i of A^{k+1} is row i of A^k (x) A (P:83 with Thm 1), and A — the right
operand of every step — is built and packed on every rank, so ranks owning disjoint
row panels never exchange matrix data.  The one real exchange per power is the stats
vector of the fused epilogue (diag min, per-alpha lo / -hi / -mis / -fin), which is
MIN-reducible by construction: one ``all_reduce(MIN)`` of 1 + 4*alpha_max int32 (<= 164 B
at alpha_max = 10), after which every rank takes the same decision (Alg 2 step 4,
P:292; first detection stops all ranks — Lemma 2).

torch.distributed is the plumbing (NCCL over NVLink on GPUs, gloo in the CPU tests);
the arithmetic runs in librd.so.
"""
from __future__ import annotations

import numpy as np

TILE = 128


def panel_bounds(N: int, world: int, rank: int, tile: int = TILE):
    """Contiguous [begin, end) rows of whole `tile`-row tiles, balanced to within one tile;
    ranks beyond the tile count get an empty panel (begin == end)."""
    ntiles = (N + tile - 1) // tile
    base, extra = divmod(ntiles, world)
    t0 = rank * base + min(rank, extra)
    t1 = t0 + base + (1 if rank < extra else 0)
    return min(N, t0 * tile), min(N, t1 * tile)


def neutral_stats(alpha_max: int) -> np.ndarray:
    """Stats of an empty panel: the identity of the elementwise MIN."""
    s = np.zeros(1 + 4 * alpha_max, dtype=np.int32)
    s[0] = 2**31 - 1
    for a in range(alpha_max):
        s[1 + 4 * a] = 2**31 - 1
        s[2 + 4 * a] = 2**31 - 1
    return s


class Decider:
    """Algorithm 2 step 4 on the reduced stats of successive powers, shared by every
    driver: feed(k, stats) records diag[k] (Cor 7) and returns True once the sequence can stop
    — at the first detection under policy 0 (Lemma 2), or once A^{n0+alpha_max} is
    seen under policy 1 (the largest alpha <= alpha_max with A^{n0+alpha} = beta (x) A^{n0}).
    Same decisions as rd_power_sequence_ex (R6)."""

    def __init__(self, alpha_max: int, policy: int, kmax: int, diag1: int):
        self.alpha_max, self.policy, self.kmax = alpha_max, policy, kmax
        self.diag = [2**31 - 1] * (kmax + 1)
        self.diag[1] = diag1
        self.found_k, self.n0, self.alpha, self.beta, self.k_stop = -1, 0, 0, 0, 1

    def feed(self, k: int, h) -> bool:
        from . import RD_INF, rd_stats_decide
        self.k_stop = k
        self.diag[k] = int(h[0]) if h[0] < RD_INF else 2**31 - 1
        if self.found_k < 0:
            dec = rd_stats_decide(h, self.alpha_max, k)
            if dec:
                self.found_k, self.n0, self.alpha, self.beta = k, k - dec[0], dec[0], dec[1]
                return self.policy == 0
            return False
        aa = k - self.n0
        if aa <= self.alpha_max:
            dec = rd_stats_decide(h, self.alpha_max, k, only_alpha=aa)
            if dec:
                self.alpha, self.beta = dec
        return aa >= self.alpha_max

    @property
    def complete(self) -> bool:
        return self.found_k >= 0 and (self.policy == 0 or self.k_stop - self.n0 >= self.alpha_max)

    def result(self, **extra) -> dict:
        return dict(found=self.found_k >= 0, n0=self.n0, alpha=self.alpha, beta=self.beta,
                    k_stop=self.k_stop, diag=self.diag, **extra)


class _EmptyPanel:
    """A rank without rows (more ranks than row tiles) still joins every collective."""

    diag1 = 2**31 - 1

    def __init__(self, alpha_max: int, device):
        import torch
        self.alpha_max = alpha_max
        self.k = 1
        self.stats = torch.from_numpy(neutral_stats(alpha_max)).to(device)

    def step(self, stats=None):
        import torch
        self.k += 1
        s = self.stats if stats is None else stats
        s.copy_(torch.from_numpy(neutral_stats(self.alpha_max)))
        return s

    def close(self):
        pass


def broadcast_chain(m: int, alpha_max: int, r0: int, r1: int, group=None, src: int = 0):
    """Dense panel chain whose packed operand is built once on rank `src` and broadcast
    (NCCL over NVLink; 969 MB at m = 9) instead of being rebuilt from the host on every
    rank.  Every rank must call it (also ranks with empty panels, which get None)."""
    import torch
    import torch.distributed as dist

    from . import Chain, count_words
    rank = dist.get_rank(group)
    N = count_words(m)
    P = (N + TILE - 1) // TILE * TILE
    words = P // 2 * P
    dev = torch.device("cuda", torch.cuda.current_device())
    if rank == src:
        # src builds a full chain over its own panel (or a 1-row one if its panel is empty)
        a, b = (r0, r1) if r1 > r0 else (0, 1)
        own = Chain(m, alpha_max=alpha_max, row_begin=a, row_end=b)
        buf = own.packed_operand()
        d1 = own.diag1 if r1 > r0 else 2**31 - 1
    else:
        own = None
        buf = torch.empty(words, dtype=torch.int32, device=dev)
        d1 = 2**31 - 1
    torch.cuda.synchronize()
    dist.broadcast(buf, src=src, group=group)
    if rank == src:
        chain = own if r1 > r0 else None
        if chain is None:
            torch.cuda.synchronize()       # the broadcast has read the buffer
            own.close()
        return chain
    if r1 <= r0:
        return None
    # this rank's diag1 from its rows of A: the packed operand holds them
    chain = Chain(m, alpha_max=alpha_max, row_begin=r0, row_end=r1, packed=buf, diag1=None)
    del buf
    return chain


def power_sequence(m: int, kmax: int = 50, alpha_max: int = 10, policy: int = 0, group=None,
                   chain_factory=None, diag1=None, method: int = 0, broadcast: bool = False):
    """Algorithm 2 over all ranks of `group`; every rank returns the same
    dict(found, n0, alpha, beta, k_stop, diag) as rd_power_sequence.

    chain_factory(m, alpha_max, row_begin, row_end) -> object with .step() returning the
    panel's stats tensor (default: paper_2409_17658_b200.Chain on the current GPU);
    diag1 = min_p A_pp (default: from rd_build_matrix).
    """
    import time

    import torch
    import torch.distributed as dist

    from . import count_words, rd_stats_decide, RD_INF

    t0 = time.perf_counter()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    N = count_words(m)
    r0, r1 = panel_bounds(N, world, rank)
    if chain_factory is None:
        from . import Chain

        def chain_factory(m_, am_, a_, b_):
            return Chain(m_, alpha_max=am_, row_begin=a_, row_end=b_, method=method)
    device = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else torch.device("cpu")
    if broadcast and world > 1 and method == 0:
        chain = broadcast_chain(m, alpha_max, r0, r1, group)
        chain = chain if chain is not None else _EmptyPanel(alpha_max, device)
    else:
        chain = chain_factory(m, alpha_max, r0, r1) if r1 > r0 else _EmptyPanel(alpha_max, device)
    if diag1 is None:
        d1 = getattr(chain, "diag1", 2**31 - 1)
        if world > 1:
            t = torch.tensor([d1], dtype=torch.int64, device=device)
            dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
            d1 = int(t.item())
        diag1 = d1

    if torch.cuda.is_available():
        torch.cuda.synchronize()
    t1 = time.perf_counter()
    dec = Decider(alpha_max, policy, kmax, diag1)
    for k in range(2, kmax + 1):
        s = chain.step()
        if world > 1:
            dist.all_reduce(s, op=dist.ReduceOp.MIN, group=group)
        if dec.feed(k, s.cpu().numpy()):
            break
    t2 = time.perf_counter()
    chain.close()
    return dec.result(t_build=t1 - t0, t_chain=t2 - t1)


# ----------------------------------------------------------- all-gather form --
def minplus_mul_allgather(A_rows, B_panel, k_bounds, group=None, acc=None):
    """Generic distributed product (the north star's all-gather form).

    Rank r holds A_rows = A[R_r, :] (M_r x K) and B_panel = B[K_r, :] (its k-rows); it
    returns C[R_r, :] = A[R_r, :] (x) B.  B's panels travel around a ring of P2P
    transfers (NCCL on GPUs): at step t the rank multiplies the panel of rank r - t into
    C (C = min(C, A[:, K_{r-t}] (x) B[K_{r-t}, :]), rd_minplus_mul_acc) while the panel of
    rank r - t - 1 is in flight, so the gather overlaps the product chunk by chunk.
    k_bounds[s] = (k0, k1) of rank s.  acc(A_rows, k0, k1, chunk, C) overrides the
    accumulating product (CPU tests use an oracle-backed one).
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    M, K = A_rows.shape
    N = B_panel.shape[1]
    from . import RD_INF
    if acc is None:
        from . import rd_minplus_mul_acc

        def acc(A_, k0, k1, chunk, C_):
            if k1 > k0 and M > 0:
                rd_minplus_mul_acc(A_, K, chunk, N, C_, N, M, N, k1 - k0, a_offset=k0)
    C = torch.full((M, N), RD_INF, dtype=torch.int16, device=A_rows.device)
    kmax_rows = max(k1 - k0 for k0, k1 in k_bounds)
    cur = torch.empty((kmax_rows, N), dtype=B_panel.dtype, device=B_panel.device)
    cur[:B_panel.shape[0]].copy_(B_panel)
    nxt = torch.empty_like(cur)
    # gloo cannot send from device memory: stage the ring through host buffers then (tests
    # run several ranks on one GPU that way); NCCL moves device buffers over NVLink directly
    staged = world > 1 and cur.is_cuda and dist.get_backend(group) == "gloo"
    if staged:
        h_cur = torch.empty(cur.shape, dtype=cur.dtype, pin_memory=True)
        h_nxt = torch.empty_like(h_cur)
    for t in range(world):
        src = (rank - t) % world
        reqs = []
        if t < world - 1:
            if staged:
                h_cur.copy_(cur)
                s_buf, r_buf = h_cur, h_nxt
            else:
                s_buf, r_buf = cur, nxt
            ops = [dist.P2POp(dist.isend, s_buf, (rank + 1) % world, group),
                   dist.P2POp(dist.irecv, r_buf, (rank - 1) % world, group)]
            reqs = dist.batch_isend_irecv(ops)
        k0, k1 = k_bounds[src]
        acc(A_rows, k0, k1, cur[:k1 - k0], C)
        for q in reqs:
            q.wait()
        if staged and t < world - 1:
            nxt.copy_(h_nxt)
        cur, nxt = nxt, cur
    return C


def power_sequence_allgather(m: int, kmax: int = 50, alpha_max: int = 10, policy: int = 0, group=None,
                             acc=None, stats=None, A=None):
    """Algorithm 2 with the left-multiplied step A^{k+1} = A (x) A^k (powers of A commute):
    rank r keeps the fixed panel A[R_r, :] and computes rows R_r of every power, gathering
    all of A^k each step through minplus_mul_allgather.  Stats of the own rows against the
    own rows of the previous powers (rd_panel_stats), all_reduce(MIN), shared decision.
    Same result dict as power_sequence.  acc / stats override the device ops (CPU tests);
    A (host int16 matrix, RD_INF = inf) skips the host build."""
    import time

    import torch
    import torch.distributed as dist

    from . import RD_INF, count_words, rd_stats_decide, rd_build_matrix

    t0 = time.perf_counter()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    N = count_words(m)
    bounds = [panel_bounds(N, world, s) for s in range(world)]
    r0, r1 = bounds[rank]
    if A is None:
        A = rd_build_matrix(m)
    on_gpu = acc is None
    device = torch.device("cuda", torch.cuda.current_device()) if on_gpu else torch.device("cpu")
    A_rows = torch.from_numpy(np.ascontiguousarray(A[r0:r1])).to(device)
    if stats is None:
        from . import rd_panel_stats, rd_stats_len
        sbuf = torch.empty(rd_stats_len(alpha_max), dtype=torch.int32, device=device)

        def stats(cur, prevs):
            return rd_panel_stats(cur, prevs, r0, alpha_max, sbuf)
    # diag[1] = min_p (A^1)_pp over this rank's rows (Cor 7 at k = 1): the stats kernel's
    # diagonal min of the panel with no earlier power
    d1 = 2**31 - 1
    if r1 > r0:
        d1 = int(stats(A_rows, []).cpu()[0])
        if d1 >= RD_INF:
            d1 = 2**31 - 1
    if world > 1:
        tt = torch.tensor([d1], dtype=torch.int64, device=device)
        dist.all_reduce(tt, op=dist.ReduceOp.MIN, group=group)
        d1 = int(tt.item())
    ring = {1: A_rows.clone()}
    if on_gpu:
        torch.cuda.synchronize()
    t1 = time.perf_counter()
    dec = Decider(alpha_max, policy, kmax, d1)
    for k in range(2, kmax + 1):
        Xk = minplus_mul_allgather(A_rows, ring[k - 1], bounds, group, acc=acc)
        ring[k] = Xk
        prevs = [ring[k - a] for a in range(1, min(alpha_max, k - 1) + 1)]
        s = stats(Xk, prevs)
        if world > 1:
            dist.all_reduce(s, op=dist.ReduceOp.MIN, group=group)
        ring.pop(k - alpha_max - 1, None)
        if dec.feed(k, s.cpu().numpy()):
            break
    t2 = time.perf_counter()
    return dec.result(t_build=t1 - t0, t_chain=t2 - t1)


# ------------------------------------------------- peer all-gather form (fused) --
def peer_bounds(N: int, world: int):
    """Row boundaries [b_0 = 0, b_1, ..., b_world = N] of the peer all-gather form: whole
    128-row tiles, balanced within one tile, every panel non-empty."""
    b = [panel_bounds(N, world, s)[0] for s in range(world)] + [N]
    if any(b[s + 1] <= b[s] for s in range(world)):
        raise ValueError(f"N={N} has fewer 128-row tiles than the {world} ranks")
    return b


def peer_chain(m: int, alpha_max: int = 10, group=None, stream=None, factory=None):
    """This rank's AgChain with every peer's ring registered: the IPC handles (64 B each) and
    slot sizes are exchanged with all_gather_object; every rank must call it.  `factory(m,
    bounds, rank, alpha_max)` overrides the chain (CPU tests)."""
    import torch.distributed as dist

    from . import AgChain, count_words
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    bounds = peer_bounds(count_words(m), world)
    if factory is None:
        chain = AgChain(m, bounds, rank, alpha_max=alpha_max, stream=stream)
    else:
        chain = factory(m, bounds, rank, alpha_max)
    if world > 1:
        info = [None] * world
        dist.all_gather_object(info, chain.ipc_handle(), group=group)
        for s in range(world):
            if s != rank:
                chain.set_peer(s, handle=info[s][0], slot_words=info[s][1])
    return chain


def power_sequence_peer(m: int, kmax: int = 50, alpha_max: int = 10, policy: int = 0, group=None,
                        factory=None):
    """Algorithm 2 in the peer all-gather form (rd_agchain): rank r
    computes rows R_r of A^{k+1} = A (x) A^k with the GEMM reading A^k from every rank's ring
    (NVLink peer memory via CUDA IPC).  The stats all_reduce(MIN) of step k is the only
    synchronisation and orders all ranks' step k before any step k+1.  Same result dict as
    power_sequence."""
    import time

    import torch
    import torch.distributed as dist

    t0 = time.perf_counter()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    on_gpu = factory is None
    device = torch.device("cuda", torch.cuda.current_device()) if on_gpu else torch.device("cpu")
    chain = peer_chain(m, alpha_max, group, factory=factory)
    d1 = chain.diag1
    if world > 1:
        t = torch.tensor([d1], dtype=torch.int64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
        d1 = int(t.item())
    if on_gpu:
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier(group=group)    # every peer mapped before any rank reads peer memory
    t1 = time.perf_counter()
    dec = Decider(alpha_max, policy, kmax, d1)
    for k in range(2, kmax + 1):
        s = chain.step()
        if world > 1:
            dist.all_reduce(s, op=dist.ReduceOp.MIN, group=group)
        if dec.feed(k, s.cpu().numpy()):
            break
    t2 = time.perf_counter()
    if world > 1:
        dist.barrier(group=group)    # no rank frees its ring while a peer may still map it
    chain.close()
    return dec.result(t_build=t1 - t0, t_chain=t2 - t1)


# ------------------------------------------- panel-sequential (one GPU or several ranks) --
def power_sequence_panels(m: int, kmax: int, alpha_max: int = 5, panel_rows: int | None = None, method: int = 1,
                          policy: int = 0, progress=None, early_stop: bool = True, group=None,
                          chain_factory=None):
    """Algorithm 2 for orders whose ring of powers does not fit one GPU (m = 11: 73 GB per
    int16 power).  Rows of A^{k+1} depend only on the same rows of A^k, so the chain
    runs panel by panel, each panel's per-power stats vector is kept, and the decision (first
    k with a uniform alpha, Alg 2 step 4) is taken on the MIN-combined stats afterwards — the
    same decision the row-panel driver takes across ranks.

    Under torch.distributed (group), rank r runs panels r, r + world, ... of the same split;
    the per-power stats arrays are MIN-reduced over the ranks (one all_reduce of
    (kend - 1) x (1 + 4 alpha_max) int32 at the end) before the shared decision.

    early_stop: each rank's first panel runs to its own first detection plus a margin (4
    powers, or alpha_max under policy 1); the ranks agree on the largest such power (MAX
    all_reduce) and every panel runs to it.  Combining panels can only delay a detection (MIN
    of the stats never creates uniformity), so if the combined decision is not reached there,
    everything is recomputed to kmax.  Returns the dict of power_sequence plus per-panel
    timings (this rank's panels).

    chain_factory(m, alpha_max, r0, r1) -> object with step() (stats tensor), diag1, close()
    (default: paper_2409_17658_b200.Chain with `method`; CPU tests pass an oracle panel)."""
    import time

    import torch
    import torch.distributed as dist

    from . import count_words, rd_stats_decide
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    N = count_words(m)
    if panel_rows is None:
        panel_rows = N
    panel_rows = max(TILE, (panel_rows + TILE - 1) // TILE * TILE)
    bounds = [(r0, min(N, r0 + panel_rows)) for r0 in range(0, N, panel_rows)]
    mine = bounds[rank::world]
    margin = alpha_max if policy == 1 else 4
    on_gpu = chain_factory is None and torch.cuda.is_available()
    device = torch.device("cuda", torch.cuda.current_device()) if on_gpu else torch.device("cpu")
    if chain_factory is None:
        from . import Chain

        def chain_factory(m_, am_, a_, b_):
            return Chain(m_, alpha_max=am_, row_begin=a_, row_end=b_, method=method)

    def sync():
        if on_gpu:
            torch.cuda.synchronize()

    def start(r0, r1):
        t0 = time.perf_counter()
        ch = chain_factory(m, alpha_max, r0, r1)
        sync()
        return {"ch": ch, "rows": [], "k": 1, "r": (r0, r1), "t0": t0, "tb": time.perf_counter() - t0}

    def advance(pn, k_to, stop_on_detect):
        seen = False
        while pn["k"] < k_to:
            k = pn["k"] + 1
            pn["rows"].append(pn["ch"].step().clone())
            pn["k"] = k
            if stop_on_detect and not seen and rd_stats_decide(pn["rows"][-1].cpu().numpy(), alpha_max, k):
                seen, k_to = True, min(k_to, k + margin)
        return pn["k"]

    def finish(pn, timings):
        st = torch.stack(pn["rows"]).cpu().numpy()
        d1 = pn["ch"].diag1
        pn["ch"].close()
        sync()
        t = {"rows": list(pn["r"]), "k_end": pn["k"], "build_s": round(pn["tb"], 3),
             "chain_s": round(time.perf_counter() - pn["t0"] - pn["tb"], 3)}
        timings.append(t)
        if progress:
            progress(t)
        return st, d1

    def allreduce(x, op):
        if world == 1:
            return x
        t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.int64)).to(device)
        dist.all_reduce(t, op=op, group=group)
        return t.cpu().numpy()

    def decide(combined, kend, diag1):
        dec = Decider(alpha_max, policy, kmax, diag1)
        for k in range(2, kend + 1):
            if dec.feed(k, combined[k - 2]):
                break
        return dec

    slen = 1 + 4 * alpha_max
    for attempt in (0, 1):
        timings, diag1 = [], 2**31 - 1
        stop = early_stop and attempt == 0
        first = start(*mine[0]) if mine else None
        k_local = advance(first, kmax, stop) if first else 0
        kend = int(allreduce(np.array([k_local]), dist.ReduceOp.MAX if world > 1 else None)[0])
        combined = np.tile(neutral_stats(alpha_max).astype(np.int64), (kend - 1, 1))
        for idx, (r0, r1) in enumerate(mine):
            pn = first if idx == 0 else start(r0, r1)
            advance(pn, kend, False)
            st, d1 = finish(pn, timings)
            diag1 = min(diag1, int(d1))
            combined = np.minimum(combined, st[:kend - 1].astype(np.int64))
        combined = allreduce(combined.reshape(-1), dist.ReduceOp.MIN if world > 1 else None).reshape(kend - 1, slen)
        diag1 = int(allreduce(np.array([diag1]), dist.ReduceOp.MIN if world > 1 else None)[0])
        dec = decide(combined.astype(np.int32), kend, diag1)
        if dec.complete or kend >= kmax:
            break
    return dec.result(panels=timings)
