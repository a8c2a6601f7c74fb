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


def power_sequence(m: int, kmax: int = 50, alpha_max: int = 10, policy: int = 0, group=None,
                   chain_factory=None, diag1=None):
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
            return Chain(m_, alpha_max=am_, row_begin=a_, row_end=b_)
    device = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else torch.device("cpu")
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
    diag = [2**31 - 1] * (kmax + 1)
    diag[1] = diag1
    found_k, n0, al, be, k = -1, 0, 0, 0, 1
    for k in range(2, kmax + 1):
        s = chain.step()
        if world > 1:
            dist.all_reduce(s, op=dist.ReduceOp.MIN, group=group)
        h = s.cpu().numpy()
        diag[k] = int(h[0]) if h[0] < RD_INF else 2**31 - 1
        if found_k < 0:
            dec = rd_stats_decide(h, alpha_max, k)
            if dec:
                found_k, n0, al, be = k, k - dec[0], dec[0], dec[1]
                if policy == 0:
                    break
        else:
            aa = k - n0
            if aa <= alpha_max:
                dec = rd_stats_decide(h, alpha_max, k, only_alpha=aa)
                if dec:
                    al, be = dec
            if aa >= alpha_max:
                break
    t2 = time.perf_counter()
    chain.close()
    return dict(found=found_k >= 0, n0=n0, alpha=al, beta=be, k_stop=min(k, kmax), diag=diag,
                t_build=t1 - t0, t_chain=t2 - t1)
