"""GPU parity: the CUDA path (through the C-ABI) against the oracle, element by element.

Integer work, so the bar is bit-exact everywhere.  Infinity is
RD_INF = 0x3FFF on the product side and INT32_MAX in the oracle; the tests re-encode.
"""
import numpy as np
import pytest

import oracle as O
from rd_inputs import operand, power_like, sample_rows, sparse_like, to_inf

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2409_17658_b200 as rd  # noqa: E402

OINF = int(O.INF)
RINF = rd.RD_INF


def _gpu(X):
    return torch.from_numpy(np.ascontiguousarray(X)).cuda()


def _oracle_mul(A16, B16, transpose=False):
    A = to_inf(A16, RINF, OINF, np.int32)
    B = to_inf(B16, RINF, OINF, np.int32)
    C = O.minplus_bt(A, np.ascontiguousarray(B.T)) if transpose else O.minplus(A, B)
    return to_inf(C, OINF, RINF, np.int16)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.init()


# ------------------------------------------------------------- generic product
@pytest.mark.parametrize("N", [1, 2, 31, 32, 33, 127, 128, 129, 255, 287, 300, 848])
@pytest.mark.parametrize("inf_frac", [0.0, 0.01, 0.5, 1.0])
def test_minplus_mul_random(N, inf_frac):
    A = operand(N, N, seed=N * 7 + 1, inf_frac=inf_frac)
    B = operand(N, N, seed=N * 7 + 2, inf_frac=inf_frac)
    C = rd.rd_minplus_mul(_gpu(A), _gpu(B)).cpu().numpy()
    assert (C == _oracle_mul(A, B)).all()


def test_minplus_mul_raw_pointer_form():
    N = 200
    A, B = operand(N, N, 11), operand(N, N, 12)
    dA, dB = _gpu(A), _gpu(B)
    dC = torch.empty((N, N), dtype=torch.int16, device="cuda")
    torch.cuda.synchronize()
    rd.rd_minplus_mul_raw(dA.data_ptr(), dB.data_ptr(), dC.data_ptr(), N)
    torch.cuda.synchronize()
    assert (dC.cpu().numpy() == _oracle_mul(A, B)).all()


def test_minplus_mul_headroom_and_clamp():
    # max finite entries (RD_INF - 1) and entries above RD_INF (clamped on load)
    N = 130
    A = operand(N, N, 21, inf_frac=0.1, lo=RINF - 10, hi=RINF - 1)
    B = operand(N, N, 22, inf_frac=0.1, lo=0, hi=5)
    C = rd.rd_minplus_mul(_gpu(A), _gpu(B)).cpu().numpy()
    want = _oracle_mul(A, B)
    want[want.astype(np.int64) >= RINF] = RINF   # sums >= RD_INF saturate to +inf
    assert (C == want).all()
    A2 = A.copy(); A2[0, :] = 0x7000                # > RD_INF: treated as +inf
    C2 = rd.rd_minplus_mul(_gpu(A2), _gpu(B)).cpu().numpy()
    assert (C2[0] == RINF).all()


def test_all_inf_rows_and_columns():
    N = 257
    A = operand(N, N, 31, inf_frac=0.2, hi=50)
    B = operand(N, N, 32, inf_frac=0.2, hi=50)
    A[5, :] = RINF; A[:, 7] = RINF; B[:, 9] = RINF; B[3, :] = RINF
    C = rd.rd_minplus_mul(_gpu(A), _gpu(B)).cpu().numpy()
    assert (C == _oracle_mul(A, B)).all()
    assert (C[5] == RINF).all() and (C[:, 9] == RINF).all()


@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (5, 300, 7), (300, 5, 129), (129, 257, 1000), (1000, 33, 33)])
def test_minplus_mul_ex_rectangular_strided(M, N, K):
    A = operand(M, K + 3, 41 + M)
    B = operand(K, N + 5, 42 + N)
    dA, dB = _gpu(A), _gpu(B)
    dC = torch.full((M, N + 2), -7, dtype=torch.int16, device="cuda")
    rd.rd_minplus_mul_ex(dA, K + 3, dB, N + 5, dC, N + 2, M, N, K)
    C = dC.cpu().numpy()
    assert (C[:, :N] == _oracle_mul(A[:, :K], B[:, :N])).all()
    assert (C[:, N:] == -7).all()    # nothing written outside the N columns


def test_minplus_mul_power_like_and_sparse_operands():
    for m, N in ((7, 2507),):
        X = power_like(N, N, m, seed=5)
        B = sparse_like(N, m, seed=6)
        C = rd.rd_minplus_mul(_gpu(X), _gpu(B)).cpu().numpy()
        rows = sample_rows(N, 96, seed=7)
        want = _oracle_mul(X[rows], B, transpose=True)
        assert (C[rows] == want).all()


def test_minplus_mul_large_sampled_rows():
    # C_9-sized product at the launch shape the chain uses, sampled rows vs the oracle
    N = 21909
    A = operand(N, N, 51, inf_frac=0.01, hi=1000)
    B = operand(N, N, 52, inf_frac=0.01, hi=1000)
    C = rd.rd_minplus_mul(_gpu(A), _gpu(B))
    rows = sample_rows(N, 24, seed=53)
    got = C[torch.from_numpy(rows).cuda()].cpu().numpy()
    assert (got == _oracle_mul(A[rows], B, transpose=True)).all()


# ---------------------------------------------------------------- power chain
def _oracle_powers(m, kmax):
    return {k: to_inf(X, OINF, RINF, np.int16) for k, X in O.powers(m, kmax)}


@pytest.mark.parametrize("m", [1, 2, 3, 4, 5, 6, 7])
def test_chain_every_power_bit_exact(m):
    ref = O.power_chain(m, 50, 10, 0)
    kstop = ref["k_stop"]
    P = _oracle_powers(m, kstop)
    ch = rd.Chain(m, alpha_max=10)
    assert (ch.read_rows(1) == P[1]).all()
    for k in range(2, kstop + 1):
        s = ch.step()
        got = ch.read_rows(k)
        assert (got == P[k]).all(), (m, k)
        st = s.cpu().numpy()
        d = int(np.diag(P[k]).min())
        assert st[0] == (d if d < RINF else min(d, RINF)), (m, k)
        # every alpha's stats against the oracle's shift test
        for a in range(1, min(10, k - 1) + 1):
            b = O.shift(to_inf(P[k], RINF, OINF, np.int32), to_inf(P[k - a], RINF, OINF, np.int32))
            dec = rd.rd_stats_decide(st, 10, k, only_alpha=a)
            assert (dec[1] if dec else None) == b, (m, k, a)
    ch.close()


@pytest.mark.parametrize("m", [1, 2, 3, 4, 5, 6, 7, 8])
def test_power_sequence_matches_oracle(m):
    ref = O.power_chain(m, 50, 10, 0)
    got = rd.rd_power_sequence(m, 50)
    for key in ("found", "n0", "alpha", "beta", "k_stop"):
        assert got[key] == ref[key], (m, key)
    assert got["t_build"] > 0 and got["t_chain"] > 0          # rd_power_sequence_timed
    assert got["diag"][1:ref["k_stop"] + 1] == ref["diag"][1:ref["k_stop"] + 1]


@pytest.mark.parametrize("m", [2, 3, 4, 5, 6, 7])
def test_power_sequence_paper_compat_table2(m, golden):
    g = golden("table2_periods.json")["table2"][str(m)]
    got = rd.rd_power_sequence(m, 50, alpha_max=5, policy=1)
    assert (got["n0"], got["alpha"], got["beta"]) == tuple(g)
    ref = O.power_chain(m, 50, 5, 1)
    assert (got["n0"], got["alpha"], got["beta"], got["k_stop"]) == (ref["n0"], ref["alpha"], ref["beta"],
                                                                      ref["k_stop"])


def test_power_sequence_m9_table2_and_sampled_rows(golden):
    # full m = 9 chain on the GPU: Table 2's (22, 5, 20) and the V13/formula gammas;
    # rows of A^k sampled and recomputed by the oracle (row_k = row_{k-1} (x) A)
    got = rd.rd_power_sequence(9, 50, alpha_max=5)
    assert (got["n0"], got["alpha"], got["beta"]) == tuple(golden("table2_periods.json")["table2"]["9"])
    assert got["k_stop"] == 27
    for n in range(3, 28):
        assert got["diag"][n] == (4 * n if n % 5 == 0 else 4 * n + 2), n


def test_chain_m9_sampled_rows_bit_exact():
    m, K = 9, 6
    A = O.matrix(m)
    rows = sample_rows(A.shape[0], 6, seed=9)
    ch = rd.Chain(m, alpha_max=5)
    R = A[rows].copy()
    for k in range(2, K + 1):
        ch.step()
        R = O.minplus(R, A, skip=True)
    got = ch.read_rows(K)[rows]
    assert (got == to_inf(R, OINF, RINF, np.int16)).all()
    ch.close()


def test_row_panels_equal_full_chain():
    # multi-GPU partition emulated sequentially on one device: panels of rows give the same
    # rows and their MIN-combined stats equal the full chain's stats
    m, K = 6, 8
    full = rd.Chain(m, alpha_max=4)
    N = full.N
    cuts = [0, 100, 129, 500, N]
    panels = [rd.Chain(m, alpha_max=4, row_begin=a, row_end=b) for a, b in zip(cuts[:-1], cuts[1:])]
    for k in range(2, K + 1):
        sf = full.step().cpu().numpy()
        sp = np.min(np.stack([p.step().cpu().numpy() for p in panels]), axis=0)
        assert (sf == sp).all(), k
        fr = full.read_rows(k)
        for p, a, b in zip(panels, cuts[:-1], cuts[1:]):
            assert (p.read_rows(k) == fr[a:b]).all()


def test_roman_cylinder_formulas_with_errata():
    def f7(n):
        c = (16 * n + 4) // 5
        return c if n % 5 == 0 else c + 1

    def f8(n):
        c = (18 * n + 4) // 5
        return c if n % 5 == 0 else (c + 1 if (n % 5 in (2, 3, 4) or n == 6) else c + 2)

    for n in range(3, 120):
        assert rd.rd_roman_cylinder(7, n) == (20 if n == 6 else f7(n)), n
        assert rd.rd_roman_cylinder(8, n) == (13 if n == 3 else f8(n)), n
        assert rd.rd_roman_cylinder(1, n) == (2 * n + 2) // 3
    for n in range(3, 60):
        assert rd.rd_roman_cylinder(3, n) == O.gamma_from_chain(O.power_chain(3), n)


def test_roman_cylinder_m9_formula():
    for n in range(3, 200):
        assert rd.rd_roman_cylinder(9, n) == (4 * n if n % 5 == 0 else 4 * n + 2), n


@pytest.mark.parametrize("variant", [0, 2, 3, 4, 8])
def test_every_gemm_variant_bit_exact(variant):
    try:
        rd.rd_set_gemm_variant(variant)
        for N, f in ((1, 0.0), (129, 0.3), (300, 0.01), (1000, 0.0)):
            A = operand(N, N, 61 + N, inf_frac=f, hi=RINF - 1 if N == 129 else 1000)
            B = operand(N, N, 62 + N, inf_frac=f)
            C = rd.rd_minplus_mul(_gpu(A), _gpu(B)).cpu().numpy()
            want = _oracle_mul(A, B)
            want[want.astype(np.int64) >= RINF] = RINF
            assert (C == want).all(), (variant, N)
        ref = O.power_chain(6, 50, 10, 0)
        got = rd.rd_power_sequence(6, 50)
        assert (got["n0"], got["alpha"], got["beta"], got["k_stop"]) == (ref["n0"], ref["alpha"], ref["beta"],
                                                                          ref["k_stop"])
        assert got["diag"][1:ref["k_stop"] + 1] == ref["diag"][1:ref["k_stop"] + 1]
        P = _oracle_powers(7, 5)
        ch = rd.Chain(7, alpha_max=3)
        for _ in range(4):
            ch.step()
        assert (ch.read_rows(5) == P[5]).all()
        ch.close()
    finally:
        rd.rd_set_gemm_variant(-1)


def test_alu_probe_reports_rates():
    r = rd.rd_alu_probe()
    assert 100 < r["dpx_minplus_per_clk_sm"] < 140     # VIADDMNMX.S16x2 at half rate: 128
    assert 100 < r["mixed_minplus_per_clk_sm"] < 200   # the DPX/IMAD mix: ~142 measured
    assert r["sm_mhz"] > 500


# ------------------------------------------------ all-gather form building blocks
def test_minplus_mul_acc_equals_min_of_chunk_products():
    M, N, K = 300, 257, 1000
    A = operand(M, K, 71, inf_frac=0.05)
    B = operand(K, N, 72, inf_frac=0.05)
    dA, dB = _gpu(A), _gpu(B)
    C = torch.full((M, N), RINF, dtype=torch.int16, device="cuda")
    cuts = [0, 130, 131, 600, K]
    for k0, k1 in zip(cuts[:-1], cuts[1:]):
        rd.rd_minplus_mul_acc(dA, K, dB[k0:k1].contiguous(), N, C, N, M, N, k1 - k0, a_offset=k0)
    assert (C.cpu().numpy() == _oracle_mul(A, B)).all()
    # accumulating into a non-INF C keeps the elementwise min
    C0 = operand(M, N, 73, inf_frac=0.0, hi=200)
    dC = _gpu(C0)
    rd.rd_minplus_mul_acc(dA, K, dB, N, dC, N, M, N, K)
    assert (dC.cpu().numpy() == np.minimum(C0, _oracle_mul(A, B))).all()


def test_panel_stats_against_oracle_shift():
    m, K = 5, 14
    P = _oracle_powers(m, K)
    am = 10
    cur = _gpu(P[K])
    prevs = [_gpu(P[K - a]) for a in range(1, am + 1)]
    s = torch.empty(rd.rd_stats_len(am), dtype=torch.int32, device="cuda")
    rd.rd_panel_stats(cur, prevs, 0, am, s)
    st = s.cpu().numpy()
    assert st[0] == int(np.diag(P[K]).min())
    for a in range(1, am + 1):
        b = O.shift(to_inf(P[K], RINF, OINF, np.int32), to_inf(P[K - a], RINF, OINF, np.int32))
        dec = rd.rd_stats_decide(st, am, K, only_alpha=a)
        assert (dec[1] if dec else None) == b, a
    # a row panel with a diagonal offset, and one entry flipped to INF
    X = P[K].copy()
    X[40, 7] = RINF
    s2 = rd.rd_panel_stats(_gpu(X[30:90]), [_gpu(P[K - 1][30:90])], 30, am, s).cpu().numpy()
    assert s2[0] == int(np.diag(X)[30:90].min())
    assert s2[3] == -1 and s2[4] == -1          # mismatch seen, finite pairs seen


def _stats_reference(X, prevs, diag_row0):
    """The MIN-reducible stats vector (rd.h rd_chain_step) of X against prevs, by definition."""
    X = X.astype(np.int64)
    s = [2**31 - 1]
    d = [X[i, diag_row0 + i] for i in range(X.shape[0]) if 0 <= diag_row0 + i < X.shape[1]]
    if d:
        s[0] = int(min(d))
    for P in prevs:
        P = P.astype(np.int64)
        fx, fp = X < RINF, P < RINF
        both = fx & fp
        if both.any():
            diff = X[both] - P[both]
            s += [int(diff.min()), -int(diff.max())]
        else:
            s += [2**31 - 1, 2**31 - 1]
        s += [-1 if (fx != fp).any() else 0, -1 if both.any() else 0]
    return np.array(s, dtype=np.int64)


@pytest.mark.parametrize("rows,cols,ld,nprev", [(300, 287, 287, 20), (64, 1000, 1008, 10), (5, 13, 13, 3),
                                                (257, 2048, 2048, 16), (33, 100, 100, 0), (40, 100, 103, 5),
                                                (129, 21909, 21909, 10)])
def test_panel_stats_one_pass_every_entry(rows, cols, ld, nprev):
    """rd_panel_stats (one pass over every alpha, 16 per pass; the flat streaming path for
    contiguous panels of any width, the per-row streaming path for ld % 8 == 0, the scalar path
    otherwise) equals the stats vector's definition entry by entry, with inf entries in both
    powers and a diagonal offset."""
    rng = np.random.default_rng(rows + cols + nprev)
    am = max(1, nprev)
    base = rng.integers(50, 90, size=(rows, ld)).astype(np.int16)
    X = base.copy()
    X[rng.random((rows, ld)) < 0.01] = RINF
    prevs = []
    for a in range(nprev):
        Pa = (base - (a % 3 == 0) * (2 * a)).astype(np.int16)     # some alphas uniform, some not
        if a % 4 == 1:
            Pa = Pa + rng.integers(0, 2, size=Pa.shape).astype(np.int16)
        Pa[rng.random((rows, ld)) < (0.0 if a % 2 else 0.01)] = RINF
        if a % 5 == 0:
            Pa[X == RINF] = RINF                                    # identical inf pattern
        prevs.append(Pa)
    dX = _gpu(X)
    s = torch.empty(rd.rd_stats_len(am), dtype=torch.int32, device="cuda")
    view = lambda T: T.view(-1)[: (rows - 1) * ld + cols].as_strided((rows, cols), (ld, 1))
    got = rd.rd_panel_stats(view(dX), [view(_gpu(P)) for P in prevs], 7, am, s).cpu().numpy().astype(np.int64)
    want = _stats_reference(X[:, :cols], [P[:, :cols] for P in prevs], 7)
    assert (got[:len(want)] == want).all(), (got[:len(want)], want)


@pytest.mark.parametrize("m", [3, 5, 7])
def test_power_sequence_allgather_single_rank(m):
    from paper_2409_17658_b200 import dist as rdist
    ref = O.power_chain(m, 50, 10, 0)
    got = rdist.power_sequence_allgather(m, 50, 10)
    assert (got["n0"], got["alpha"], got["beta"], got["k_stop"]) == (ref["n0"], ref["alpha"], ref["beta"],
                                                                      ref["k_stop"])
    assert got["diag"][1:ref["k_stop"] + 1] == ref["diag"][1:ref["k_stop"] + 1]


def test_power_sequence_replicated_single_rank_driver():
    from paper_2409_17658_b200 import dist as rdist
    for m in (2, 6):
        ref = O.power_chain(m, 50, 10, 0)
        got = rdist.power_sequence(m, 50, 10)
        assert (got["n0"], got["alpha"], got["beta"], got["k_stop"]) == (ref["n0"], ref["alpha"], ref["beta"],
                                                                          ref["k_stop"])


# ----------------------------------------------------- structured step (NEXT-3)
@pytest.mark.parametrize("m", [1, 2, 3, 4, 5, 6, 7])
def test_structured_chain_every_power_bit_exact(m):
    ref = O.power_chain(m, 50, 10, 0)
    kstop = ref["k_stop"]
    P = _oracle_powers(m, kstop)
    ch = rd.Chain(m, alpha_max=10, method=1)
    assert (ch.read_rows(1) == P[1]).all()
    nnz = int((P[1] < RINF).sum())
    assert ch.terms_per_step == float(P[1].shape[0]) * nnz
    for k in range(2, kstop + 1):
        st = ch.step().cpu().numpy()
        assert (ch.read_rows(k) == P[k]).all(), (m, k)
        assert st[0] == int(np.diag(P[k]).min()), (m, k)
        for a in range(1, min(10, k - 1) + 1):
            b = O.shift(to_inf(P[k], RINF, OINF, np.int32), to_inf(P[k - a], RINF, OINF, np.int32))
            dec = rd.rd_stats_decide(st, 10, k, only_alpha=a)
            assert (dec[1] if dec else None) == b, (m, k, a)
    ch.close()


@pytest.mark.parametrize("m", [1, 2, 3, 4, 5, 6, 7, 8, 9])
def test_structured_power_sequence_matches(m, golden):
    got = rd.rd_power_sequence(m, 50, method=1)
    if m <= 8:
        ref = O.power_chain(m, 50, 10, 0)
        assert (got["n0"], got["alpha"], got["beta"], got["k_stop"]) == (ref["n0"], ref["alpha"], ref["beta"],
                                                                          ref["k_stop"])
        assert got["diag"][1:ref["k_stop"] + 1] == ref["diag"][1:ref["k_stop"] + 1]
    else:
        dense = rd.rd_power_sequence(9, 50, method=0)
        assert got["diag"] == dense["diag"]
        assert (got["n0"], got["alpha"], got["beta"]) == (22, 5, 20)


def test_structured_panels_and_sampled_rows_m9():
    m, K = 9, 5
    A = O.matrix(m)
    N = A.shape[0]
    rows = sample_rows(N, 5, seed=19)
    R = A[rows].copy()
    for _ in range(2, K + 1):
        R = O.minplus(R, A, skip=True)
    R16 = to_inf(R, OINF, RINF, np.int16)
    cuts = [0, 7001, 14002, N]     # ragged panels (not multiples of 4)
    for a, b in zip(cuts[:-1], cuts[1:]):
        ch = rd.Chain(m, alpha_max=3, row_begin=a, row_end=b, method=1)
        for _ in range(K - 1):
            ch.step()
        got = ch.read_rows(K)
        sel = [r for r in rows if a <= r < b]
        assert (got[[r - a for r in sel]] == R16[[list(rows).index(r) for r in sel]]).all()
        ch.close()


# ---------------------------------------------------------------- m = 10 (NEXT-2)
def test_m10_structured_chain_pins():
    # beyond the paper ("too big"): pinned by Cor 12 (P:501-507, 5 | n, m >= 10),
    # and by the independent row DP X3 for n = 3..8
    got = rd.rd_power_sequence(10, 50, alpha_max=10, method=1)
    assert got["found"]
    d = got["diag"]
    for n in range(5, got["k_stop"] + 1, 5):
        assert d[n] == 22 * n // 5, n
    for n in range(3, 11):
        assert d[n] == O.gamma_rowdp(10, n), n
    g = O.gamma_from_chain(got, 200)
    assert g == 22 * 200 // 5                      # Cor 12 through the recurrence
    for n in range(10, 201, 5):
        assert O.gamma_from_chain(got, n) == 22 * n // 5
    for n in range(10, 201):
        assert O.gamma_from_chain(got, n) >= -(-22 * n // 5)   # Thm 11 lower bound ceil(2(m+1)n/5)


def test_m10_dense_equals_structured_first_powers():
    m, K = 10, 4
    N = rd.count_words(m)
    rows = sample_rows(N, 8, seed=23)
    outs = []
    for method in (0, 1):
        ch = rd.Chain(m, alpha_max=3, method=method)
        for _ in range(K - 1):
            ch.step()
        outs.append(ch.read_rows(K)[rows])
        ch.close()
    assert (outs[0] == outs[1]).all()
    A = O.matrix(m)
    R = A[rows].copy()
    for _ in range(K - 1):
        R = O.minplus(R, A, skip=True)
    assert (outs[1] == to_inf(R, OINF, RINF, np.int16)).all()



# ------------------------------------------------------ App. A border (NEXT-1)
@pytest.mark.parametrize("method", [0, 1])
def test_border_chain_matches_oracle(method, golden):
    A = rd.rd_build_matrix_border()
    ref = O.power_chain_matrix(O.border_matrix(), 50, 10, 0)
    got = rd.rd_power_sequence_matrix(A, 50, 10, 0, method)
    assert (got["n0"], got["alpha"], got["beta"], got["k_stop"]) == (ref["n0"], ref["alpha"], ref["beta"],
                                                                      ref["k_stop"])
    assert (got["n0"], got["alpha"], got["beta"]) == tuple(golden("border_appendix_a.json")["triple"])
    assert got["diag"][1:ref["k_stop"] + 1] == ref["diag"][1:ref["k_stop"] + 1]
    P = {k: to_inf(X, OINF, RINF, np.int16) for k, X in
         ((k, X) for k, X in _border_powers(8))}
    ch = rd.Chain(4, alpha_max=4, method=method, matrix=A)
    for k in range(2, 9):
        ch.step()
        assert (ch.read_rows(k) == P[k]).all(), k
    ch.close()


def _border_powers(kmax):
    A = O.border_matrix()
    X = A.copy()
    yield 1, X
    for k in range(2, kmax + 1):
        X = O.minplus(X, A)
        yield k, X


def test_power_sequence_matrix_random_generic():
    # a generic sparse matrix through the same pipeline (dense and structured) vs the oracle
    A16 = sparse_like(300, 6, seed=31)
    A32 = to_inf(A16, RINF, OINF, np.int32)
    ref = O.power_chain_matrix(A32, 40, 10, 0)
    for method in (0, 1):
        got = rd.rd_power_sequence_matrix(A16, 40, 10, 0, method)
        assert (got["found"], got["n0"], got["alpha"], got["beta"], got["k_stop"]) == (
            ref["found"], ref["n0"], ref["alpha"], ref["beta"], ref["k_stop"])
        assert got["diag"][1:ref["k_stop"] + 1] == ref["diag"][1:ref["k_stop"] + 1]


def test_closed_form_gpu_m9_formula():
    f = rd.rd_closed_form(9)
    assert (f["alpha"], f["beta"], f["d"], f["n_valid"]) == (5, 20, [0, 2, 2, 2, 2], 3)   # 4n / 4n+2


def test_chain_from_packed_operand_equals_built_chain():
    # the broadcast path of the row-panel driver, emulated in one process: rank 0's packed
    # operand feeds a chain for another panel, which must equal a chain built from the host
    m, K = 6, 8
    src = rd.Chain(m, alpha_max=4, row_begin=0, row_end=128)
    buf = src.packed_operand().clone()
    N = src.N
    for a, b in ((128, 700), (700, N)):
        ref = rd.Chain(m, alpha_max=4, row_begin=a, row_end=b)
        got = rd.Chain(m, alpha_max=4, row_begin=a, row_end=b, packed=buf)
        assert got.diag1 == ref.diag1
        for k in range(2, K + 1):
            s1, s2 = ref.step().cpu().numpy(), got.step().cpu().numpy()
            assert (s1 == s2).all(), k
        assert (ref.read_rows(K) == got.read_rows(K)).all()
        ref.close()
        got.close()
    src.close()


@pytest.mark.parametrize("m,r0,r1", [(6, 0, 848), (7, 0, 2507), (8, 0, 1024), (8, 3712, 4736)])
def test_split_k_equals_single_pass(m, r0, r1):
    outs = []
    rd.rd_set_stream_k(0)
    for on in (True, False):
        rd.rd_set_split_k(on)
        try:
            ch = rd.Chain(m, alpha_max=6, row_begin=r0, row_end=r1)
            st = [ch.step().cpu().numpy() for _ in range(7)]
            outs.append((st, ch.read_rows(8)))
            ch.close()
        finally:
            rd.rd_set_split_k(True)
            rd.rd_set_stream_k(0)
    for a, b in zip(outs[0][0], outs[1][0]):
        assert (a == b).all()
    assert (outs[0][1] == outs[1][1]).all()


@pytest.mark.parametrize("m,r0,r1,tn,n", [(7, 0, 2507, 128, 2), (7, 0, 2507, 64, 3), (8, 0, 1024, 128, 5),
                                         (8, 0, 1024, 64, 2)])
def test_tail_split_equals_single_pass(m, r0, r1, tn, n):
    """Tail splits (rd_set_split_tail(2): the whole waves unsplit, the last partial wave's tiles
    split n ways and finished in-kernel by their last split) give every power and stats vector of
    the plain step, and the powers equal the oracle's for m <= 7."""
    outs = []
    try:
        for tail in (True, False):
            rd.rd_set_gemm_tile(tn)
            rd.rd_set_split_tail(2 if tail else 0)
            rd.rd_set_split_k(n if tail else 0)
            if tail:
                assert rd.rd_dense_step_plan(r1 - r0, rd.count_words(m))[:3] == (tn, n, True)
            ch = rd.Chain(m, alpha_max=6, row_begin=r0, row_end=r1)
            st = [ch.step().cpu().numpy() for _ in range(2, 13)]
            outs.append((st, {k: ch.read_rows(k) for k in (8, 12)}))
            ch.close()
    finally:
        rd.rd_set_gemm_tile(0)
        rd.rd_set_split_tail(1)
        rd.rd_set_split_k(True)
    for a, b in zip(outs[0][0], outs[1][0]):
        assert (a == b).all()
    for k in outs[0][1]:
        assert (outs[0][1][k] == outs[1][1][k]).all(), k
    if m <= 7:
        P = {k: X for k, X in O.powers(m, 12) if k == 12}
        assert (outs[0][1][12] == to_inf(P[12][r0:r1], OINF, RINF, np.int16)).all()


@pytest.mark.parametrize("m,r0,r1", [(3, 0, 33), (5, 0, 287), (6, 0, 848), (7, 0, 2507), (7, 128, 1000),
                                     (8, 3712, 4736)])
def test_stream_k_equals_oracle_and_single_pass(m, r0, r1):
    """Stream-K steps with the in-kernel fixup — hybrid (rd_set_stream_k(2): the partial last
    wave's stages spread over every CTA slot) and full (3: every stage of the step) — give every
    power and every stats vector of the plain one-tile-per-CTA step, and the powers equal the
    oracle's on the full matrix for m <= 7."""
    outs = []
    rd.rd_set_split_k(False)
    try:
        for mode in (2, 3, 0):
            rd.rd_set_stream_k(mode)
            ch = rd.Chain(m, alpha_max=6, row_begin=r0, row_end=r1)
            st, rows = [], {}
            for k in range(2, 13):
                st.append(ch.step().cpu().numpy())
                if k in (2, 5, 12):
                    rows[k] = ch.read_rows(k)
            outs.append((st, rows))
            ch.close()
    finally:
        rd.rd_set_stream_k(0)
        rd.rd_set_split_k(True)
    for o in outs[:2]:
        for a, b in zip(o[0], outs[2][0]):
            assert (a == b).all()
        for k in o[1]:
            assert (o[1][k] == outs[2][1][k]).all(), k
    if m <= 7:
        P = {k: X for k, X in O.powers(m, 12) if k in (2, 5, 12)}
        for k, X in P.items():
            assert (outs[0][1][k] == to_inf(X[r0:r1], OINF, RINF, np.int16)).all(), k



@pytest.mark.parametrize("m,rows,method", [(6, 256, 1), (7, 640, 1), (7, 1024, 0)])
def test_panel_sequential_driver_matches_oracle(m, rows, method):
    from paper_2409_17658_b200 import dist as rdist
    ref = O.power_chain(m, 50, 5, 0)
    got = rdist.power_sequence_panels(m, ref["k_stop"] + 3, alpha_max=5, panel_rows=rows, method=method)
    assert len(got["panels"]) > 1
    assert (got["n0"], got["alpha"], got["beta"], got["k_stop"]) == (ref["n0"], ref["alpha"], ref["beta"],
                                                                      ref["k_stop"])
    assert got["diag"][1:ref["k_stop"] + 1] == ref["diag"][1:ref["k_stop"] + 1]



def test_m11_panel_sequential_pins():
    # m = 11 (N = 191476) on one GPU, panel by panel with the slab structured step (~50 s):
    # Cor 12 (24n/5 for 5 | n) and the independent row DP X3 for n = 3..10
    from paper_2409_17658_b200 import dist as rdist
    got = rdist.power_sequence_panels(11, 45, alpha_max=5, panel_rows=57344, method=1)
    assert got["found"]
    d = got["diag"]
    for n in range(5, got["k_stop"] + 1, 5):
        assert d[n] == 24 * n // 5, n
    for n in range(3, 11):
        assert d[n] == O.gamma_rowdp(11, n), n


@pytest.mark.parametrize("wmax,kmax", [(20, 30), (100, 12), (300, 10)])
def test_structured_byte_path_and_fallback(wmax, kmax):
    # column-uniform labels select the byte kernel; wider labels make row spreads cross 254
    # during the chain (wmax=100) or from the start (wmax=300), forcing the 16-bit kernel
    rng = np.random.default_rng(wmax)
    N = 2100                      # >= 2048: the default slab layout (smaller N take the 16-bit kernel)
    pat = rng.random((N, N)) < 0.01
    np.fill_diagonal(pat, True)
    w = rng.integers(0, wmax + 1, size=N)
    A16 = np.where(pat, w[None, :], RINF).astype(np.int16)
    A32 = to_inf(A16, RINF, OINF, np.int32)
    ch = rd.Chain(0, alpha_max=4, method=1, matrix=A16)
    X = A32.copy()
    for k in range(2, kmax + 1):
        st = ch.step().cpu().numpy()
        X = O.minplus(X, A32, skip=True)
        got = ch.read_rows(k)
        assert (got == to_inf(X, OINF, RINF, np.int16)).all(), (wmax, k)
        assert st[0] == min(int(np.diag(X).min()), RINF)
    ch.close()
    for method in (0, 1):
        got = rd.rd_power_sequence_matrix(A16, kmax, 4, 0, method)
        ref = O.power_chain_matrix(A32, kmax, 4, 0)
        assert got["diag"][1:ref["k_stop"] + 1] == ref["diag"][1:ref["k_stop"] + 1]


@pytest.mark.parametrize("m,r0,r1", [(7, 0, 2507), (8, 1000, 2999)])
def test_structured_kernel_modes_identical(m, r0, r1):
    # slab layout (2, columns permuted, stats after the product from a row sample plus full
    # passes for survivors), byte kernel (1) and 16-bit kernel (0): the same powers, diag and
    # per-alpha decisions at every power, past first detection (survivor passes run)
    outs = []
    for mode in (2, 1, 0):
        rd.rd_set_sparse_bytes(mode)
        try:
            ch = rd.Chain(m, alpha_max=6, method=1, row_begin=r0, row_end=r1)
            diag, dec, rows = [], [], []
            for k in range(2, 31):
                s = ch.step().cpu().numpy()
                diag.append(int(s[0]))
                dec.append([rd.rd_stats_decide(s, 6, k, only_alpha=a) for a in range(1, min(6, k - 1) + 1)])
                if k in (3, 9, 30):
                    rows.append(ch.read_rows(k))
            outs.append((diag, dec, rows))
            ch.close()
        finally:
            rd.rd_set_sparse_bytes(2)
    for o in outs[1:]:
        assert o[0] == outs[0][0]
        assert o[1] == outs[0][1]
        for a, b in zip(o[2], outs[0][2]):
            assert (a == b).all()
    # the decisions do detect the period (m = 7, 8: alpha = 5 at k = 26 for the full panel)
    if r0 == 0:
        assert outs[0][1][26 - 2][5 - 1] == (5, 16)


@pytest.mark.parametrize("m,method", [(8, 0), (9, 0), (9, 1)])
def test_every_power_sampled_rows_full_size(m, method):
    # rows of A^k for every k up to first detection, recomputed by the oracle's INF-skipping
    # row recurrence (row_k = row_{k-1} (x) A)
    A = O.matrix(m)
    N = A.shape[0]
    kstop = {8: 26, 9: 27}[m]
    rows = sample_rows(N, 40, seed=100 + m)
    R = A[rows].copy()
    ch = rd.Chain(m, alpha_max=10, method=method)
    for k in range(2, kstop + 1):
        ch.step()
        R = O.minplus(R, A, skip=True)
        got = ch.read_rows(k)[rows]
        assert (got == to_inf(R, OINF, RINF, np.int16)).all(), (m, k)
    ch.close()


@pytest.mark.parametrize("method", [0, 1])
def test_m8_every_power_full_matrix(method):
    """Alg 2 step 4 compares whole matrices: at m = 8 (N = 7411) every power A^k,
    k = 1..26 (first detection, Table 2), equals the oracle's X4 chain entry for entry —
    dense GEMM chain (method 0) and structured chain (method 1)."""
    ch = rd.Chain(8, alpha_max=10, method=method)
    for k, X in O.powers(8, 26):
        if k > 1:
            ch.step()
        got = ch.read_rows(k)
        assert (got == to_inf(X, OINF, RINF, np.int16)).all(), (method, k)
    ch.close()


def _digest16(X16):
    import hashlib
    return hashlib.blake2b(np.ascontiguousarray(X16.astype("<i2")).tobytes(), digest_size=8).hexdigest()


@pytest.mark.parametrize("method", [0, 1])
def test_m9_every_power_full_matrix_hash(method, golden):
    """m = 9 (N = 21909): every full power A^k, k = 1..27 (k* of Table 2), hashed (BLAKE2b-64 of
    the row-major int16 matrix, inf = 0x3FFF) equals the digest of the oracle's X4 chain written
    by tools/make_golden.py (oracle only) — plus its inf count and diagonal min."""
    g = golden("m9_power_hashes.json")
    assert g["N"] == 21909 and g["kmax"] == 27
    ch = rd.Chain(9, alpha_max=2, method=method)
    for k in range(1, 28):
        if k > 1:
            s = ch.step().cpu().numpy()
            assert int(s[0]) == g["powers"][str(k)]["diag_min"], k
        X = ch.read_rows(k)
        want = g["powers"][str(k)]
        assert int((X == RINF).sum()) == want["n_inf"], (method, k)
        assert _digest16(X) == want["blake2b64"], (method, k)
    ch.close()


def test_border_n11_erratum_on_gpu(golden):
    """P:664 claims 2 L_a(n) = n for 10 <= n <= 30; at n = 11 the library's border chain
    (App. A matrix, dense and structured) gives the oracle row DP's value written by
    tools/make_golden.py (12, R16)."""
    want = golden("border_n11_rowdp.json")
    assert want["n"] == 11 and want["value"] == 12
    A = rd.rd_build_matrix_border()
    for method in (0, 1):
        got = rd.rd_power_sequence_matrix(A, 50, 10, 0, method)
        assert got["diag"][11] == want["value"]
        for n in range(10, 31):
            if n != 11:
                assert got["diag"][n] == n if n <= got["k_stop"] else True


def test_device_allocation_failure_is_reported():
    # a dense m = 11 chain with a 33-power ring needs ~2.4 TB: RD_ENOMEM from the device-memory
    # check before any host build (fast), no crash, and the device stays usable
    import time
    t0 = time.perf_counter()
    with pytest.raises(rd.RDError) as e:
        rd.Chain(11, alpha_max=32)
    assert e.value.status == rd.RD_ENOMEM and "GB free" in str(e.value)
    assert time.perf_counter() - t0 < 5.0
    with pytest.raises(rd.RDError) as e:
        rd.Chain(3, alpha_max=17, method=1)          # structured step: alpha_max <= 16
    assert e.value.status == rd.RD_EINVAL
    C = rd.rd_minplus_mul(_gpu(operand(64, 64, 1)), _gpu(operand(64, 64, 2)))
    assert C.shape == (64, 64)


# ------------------------------------------------ peer all-gather chain (fused) --
@pytest.mark.parametrize("m", [1, 3, 5, 7])
def test_agchain_single_rank_every_power_bit_exact(m):
    # A^{k+1} = A (x) A^k with the right operand read through the peer table (one rank):
    # every power and every alpha's stats against the oracle (Alg 2 step 4)
    ref = O.power_chain(m, 50, 10, 0)
    kstop = ref["k_stop"]
    P = _oracle_powers(m, kstop)
    N = P[1].shape[0]
    ch = rd.AgChain(m, [0, N], 0, alpha_max=10)
    assert (ch.read_rows(1) == P[1]).all()
    for k in range(2, kstop + 1):
        st = ch.step().cpu().numpy()
        assert (ch.read_rows(k) == P[k]).all(), (m, k)
        d = int(np.diag(P[k]).min())
        assert st[0] == min(d, RINF), (m, k)
        for a in range(1, min(10, k - 1) + 1):
            b = O.shift(to_inf(P[k], RINF, OINF, np.int32), to_inf(P[k - a], RINF, OINF, np.int32))
            dec = rd.rd_stats_decide(st, 10, k, only_alpha=a)
            assert (dec[1] if dec else None) == b, (m, k, a)
    ch.close()


@pytest.mark.parametrize("m,cuts", [(5, [0, 128, 287]), (6, [0, 256, 384, 848]),
                                    (7, [0, 640, 1280, 1920, 2507])])
def test_agchain_panels_in_process_equal_full_chain(m, cuts):
    # several ranks emulated in one process on one device: each panel's GEMM reads the other
    # panels' ring slots through device pointers (the IPC path maps the same layout); steps
    # are separated by a device sync, as the stats all_reduce separates them across GPUs
    K = 9
    full = rd.Chain(m, alpha_max=4)
    ranks = [rd.AgChain(m, cuts, r, alpha_max=4) for r in range(len(cuts) - 1)]
    for r, c in enumerate(ranks):
        for s, o in enumerate(ranks):
            if s != r:
                ptr, words = o.ring()
                c.set_peer(s, ring_ptr=ptr, slot_words=words)
    for k in range(2, K + 1):
        sf = full.step().cpu().numpy()
        sp = [c.step(torch.empty_like(c.stats)) for c in ranks]
        torch.cuda.synchronize()
        sp = np.min(np.stack([x.cpu().numpy() for x in sp]), axis=0)
        assert (sf == sp).all(), (m, k)
        fr = full.read_rows(k)
        for c, a, b in zip(ranks, cuts[:-1], cuts[1:]):
            assert (c.read_rows(k) == fr[a:b]).all(), (m, k, a)
    for c in ranks:
        c.close()
    full.close()


@pytest.mark.parametrize("m", [4, 7, 8])
def test_power_sequence_peer_single_rank(m):
    from paper_2409_17658_b200 import dist as rdist
    ref = O.power_chain(m, 50, 10, 0)
    got = rdist.power_sequence_peer(m, 50, 10)
    assert (got["n0"], got["alpha"], got["beta"], got["k_stop"]) == (ref["n0"], ref["alpha"], ref["beta"],
                                                                      ref["k_stop"])
    assert got["diag"][1:ref["k_stop"] + 1] == ref["diag"][1:ref["k_stop"] + 1]


def test_agchain_bad_arguments():
    N = rd.count_words(5)
    with pytest.raises(rd.RDError):
        rd.AgChain(5, [0, 100, N], 0)          # panel 1 does not start on a 128-row tile
    with pytest.raises(rd.RDError):
        rd.AgChain(5, [0, N - 1], 0)           # bounds must end at N
    c = rd.AgChain(5, [0, 128, N], 0)
    with pytest.raises(rd.RDError):
        c.step()                               # rank 1's ring not registered
    with pytest.raises(rd.RDError):
        c.set_peer(1, ring_ptr=c.ring()[0], slot_words=7)   # wrong slot size
    c.close()


def test_agchain_m9_every_power_sampled_rows_and_detection():
    # the peer all-gather form at the bench's full size (m = 9, world 1, the launch bench.py
    # --form peer times): sampled rows of every power to first detection against the oracle's
    # row recurrence, and the stats decision (22, 5, 20) at k = 27 (Table 2)
    m = 9
    A = O.matrix(m)
    N = A.shape[0]
    rows = sample_rows(N, 24, seed=309)
    R = A[rows].copy()
    ch = rd.AgChain(m, [0, N], 0, alpha_max=10)
    dec = None
    for k in range(2, 28):
        st = ch.step().cpu().numpy()
        R = O.minplus(R, A, skip=True)
        assert (ch.read_rows(k)[rows] == to_inf(R, OINF, RINF, np.int16)).all(), k
        d = rd.rd_stats_decide(st, 10, k)
        if dec is None and d:
            dec = (k, k - d[0], d[0], d[1])
    assert dec == (27, 22, 5, 20)
    ch.close()


# ------------------------------------------------------ 32-bit generic product --
RINF32 = rd.RD_INF32


def _oracle_mul32(A32, B32):
    A = to_inf(A32, RINF32, OINF, np.int32)
    B = to_inf(B32, RINF32, OINF, np.int32)
    return to_inf(O.minplus(A, B), OINF, RINF32, np.int32)


@pytest.mark.parametrize("N", [1, 33, 129, 300, 1000])
@pytest.mark.parametrize("inf_frac", [0.0, 0.05, 1.0])
def test_minplus_mul32_random(N, inf_frac):
    # values far beyond the int16 headroom (up to 2^29 - 1): exact against the oracle
    A = operand(N, N, seed=N * 11 + 1, inf_frac=inf_frac, hi=2**29 - 1, inf=RINF32, dtype=np.int32)
    B = operand(N, N, seed=N * 11 + 2, inf_frac=inf_frac, hi=2**29 - 1, inf=RINF32, dtype=np.int32)
    C = rd.rd_minplus_mul32(_gpu(A), _gpu(B)).cpu().numpy()
    assert (C == _oracle_mul32(A, B)).all()


@pytest.mark.parametrize("M,N,K", [(5, 300, 7), (300, 5, 129), (129, 257, 1000), (1000, 33, 31)])
def test_minplus_mul32_rectangular(M, N, K):
    A = operand(M, K, seed=M + K, inf_frac=0.1, hi=10**6, inf=RINF32, dtype=np.int32)
    B = operand(K, N, seed=N + K, inf_frac=0.1, hi=10**6, inf=RINF32, dtype=np.int32)
    C = rd.rd_minplus_mul32(_gpu(A), _gpu(B)).cpu().numpy()
    assert (C == _oracle_mul32(A, B)).all()


def test_minplus_mul32_saturation_and_clamp():
    # finite sums >= RD_INF32 saturate to RD_INF32 (rd.h); inputs above RD_INF32 clamp to it
    N = 130
    A = operand(N, N, 41, inf_frac=0.1, lo=2**29, hi=RINF32 - 1, inf=RINF32, dtype=np.int32)
    B = operand(N, N, 42, inf_frac=0.1, lo=0, hi=2**29 + 5, inf=2**31 - 1, dtype=np.int32)
    C = rd.rd_minplus_mul32(_gpu(A), _gpu(B)).cpu().numpy()
    Bc = np.minimum(B, RINF32)
    want = np.minimum(_oracle_mul32(A, Bc).astype(np.int64), RINF32).astype(np.int32)
    assert (C == want).all()


@pytest.mark.parametrize("variant", [0, 2, 3, 4, 8])
def test_minplus_mul32_every_variant_and_int16_agreement(variant):
    # every mainloop mix is bit-identical; on int16-range data the 32-bit product equals the
    # 16-bit one (infinities mapped)
    N = 257
    A16 = operand(N, N, 51, inf_frac=0.02, hi=5000)
    B16 = operand(N, N, 52, inf_frac=0.02, hi=5000)
    try:
        rd.rd_set_gemm_variant(variant)
        C32 = rd.rd_minplus_mul32(_gpu(to_inf(A16, RINF, RINF32, np.int32)),
                                  _gpu(to_inf(B16, RINF, RINF32, np.int32))).cpu().numpy()
        C16 = rd.rd_minplus_mul(_gpu(A16), _gpu(B16)).cpu().numpy()
    finally:
        rd.rd_set_gemm_variant(-1)
    assert (C32 == to_inf(C16, RINF, RINF32, np.int32)).all()
    assert (C32 == _oracle_mul32(to_inf(A16, RINF, RINF32, np.int32), to_inf(B16, RINF, RINF32, np.int32))).all()


@pytest.mark.parametrize("M,N,K", [(7, 130, 33), (129, 5, 300)])
def test_minplus_mul32_ex_strided_guard(M, N, K):
    # leading dimensions larger than the shapes; nothing written outside the N columns of C
    A = operand(M, K + 3, 61 + M, inf_frac=0.05, hi=2**28, inf=RINF32, dtype=np.int32)
    B = operand(K, N + 5, 62 + N, inf_frac=0.05, hi=2**28, inf=RINF32, dtype=np.int32)
    dA, dB = _gpu(A), _gpu(B)
    dC = torch.full((M, N + 2), -7, dtype=torch.int32, device="cuda")
    rc = rd.lib().rd_minplus_mul32_ex(dA.data_ptr(), K + 3, dB.data_ptr(), N + 5, dC.data_ptr(), N + 2, M, N, K,
                                      None)
    assert rc == rd.RD_OK
    C = dC.cpu().numpy()
    assert (C[:, :N] == _oracle_mul32(np.ascontiguousarray(A[:, :K]), np.ascontiguousarray(B[:, :N]))).all()
    assert (C[:, N:] == -7).all()


def test_minplus_mul32_large_sampled_rows():
    # the 32-bit product at a bench-like size (N = 7411, uniform [0, 2^29), 1% inf): sampled
    # output rows recomputed by the oracle through B's transpose
    N = 7411
    A = operand(N, N, 71, inf_frac=0.01, hi=2**29 - 1, inf=RINF32, dtype=np.int32)
    B = operand(N, N, 72, inf_frac=0.01, hi=2**29 - 1, inf=RINF32, dtype=np.int32)
    C = rd.rd_minplus_mul32(_gpu(A), _gpu(B)).cpu().numpy()
    rows = sample_rows(N, 12, seed=73)
    Ao = to_inf(A[rows], RINF32, OINF, np.int32)
    BT = np.ascontiguousarray(to_inf(B, RINF32, OINF, np.int32).T)
    want = to_inf(O.minplus_bt(Ao, BT), OINF, RINF32, np.int32)
    assert (C[rows] == want).all()


@pytest.mark.parametrize("m,r0,r1,tile", [(6, 0, 848, 0), (7, 0, 2507, 0), (8, 1000, 2999, 0), (7, 0, 2507, 128),
                                          (8, 0, 1024, 128), (8, 0, 7411, 128)])
def test_tma_mainloop_bit_identical(m, r0, r1, tile):
    # the TMA + mbarrier mainloop (forced on, incl. uniform and tail split-K steps: the 128-wide
    # plans of m = 7 / 8) = the cp.async mainloop, powers and stats, for whole and partial panels
    def run(mode):
        rd.rd_set_gemm_tma(mode)
        rd.rd_set_gemm_tile(tile)
        try:
            ch = rd.Chain(m, alpha_max=6, row_begin=r0, row_end=r1)
            st = [ch.step().cpu().numpy().copy() for _ in range(7)]
            rows = ch.read_rows(ch.k)
            ch.close()
        finally:
            rd.rd_set_gemm_tma(1)
            rd.rd_set_gemm_tile(0)
        return np.stack(st), rows
    s0, x0 = run(0)
    s2, x2 = run(2)
    assert (s0 == s2).all() and (x0 == x2).all()


@pytest.mark.parametrize("m,method", [(8, 0), (8, 1), (9, 0), (9, 1)])
def test_v24_checksums_full_size(m, method, golden):
    # every entry of A^1..A^5 at the full m = 8 / m = 9 size, through word-order-invariant sums
    # (#inf, sum of finite entries, sum of the finite diagonal) produced at survey time by an
    # independent model (tests/golden/survey_checksums_v24.json)
    want = golden("survey_checksums_v24.json")["checksums"][str(m)]
    ch = rd.Chain(m, alpha_max=5, method=method)
    for k in range(1, 6):
        if k > 1:
            ch.step()
        if str(k) not in want:
            continue
        X = ch.read_rows(k)
        fin = X < RINF
        got = [int((~fin).sum()), int(X[fin].astype(np.int64).sum()),
               int(np.diag(X)[np.diag(fin)].astype(np.int64).sum())]
        assert got == want[str(k)], (m, method, k)
        del X, fin
    ch.close()


def test_structured_chain_nnz_pins_m9_m10():
    # the library's CSC of A(G) has the survey's independent arc counts: nnz = 2 656 733 at m = 9
    # (V11) and 13 327 868 at m = 10 (V27); rows * nnz terms per structured step
    for m, nnz in ((9, 2656733), (10, 13327868)):
        ch = rd.Chain(m, alpha_max=5, row_begin=0, row_end=8, method=1)
        assert ch.terms_per_step == 8 * nnz, m
        ch.close()


# ------------------------------------------- orders with N >= 2^17 (q-chunked CSC) --
def _oracle_rows_a1(m, rows):
    W = O.words(m)
    out = np.full((len(rows), len(W)), rd.RD_INF, dtype=np.int16)
    for r, q in enumerate(rows):
        for p, wp in enumerate(W):
            if O.can_follow(W[q], wp):
                out[r, p] = O.label(wp)
    return out


def test_m11_operands_decode_rows_beyond_2_17():
    """m = 11 (N = 191476 >= 2^17): the CSC entries hold q - ch * Qc in 17 bits, so the operand
    scatter must decode per q-chunk; rows on both sides of 2^17 of the dense chain's A^1 panel
    (scatter_dense_operands_kernel) and of the peer chain's A^1 slot (scatter_rp_kernel) equal
    the oracle's can-follow rules and labels."""
    N = rd.count_words(11)
    assert N == 191476 > (1 << 17)
    r0 = (1 << 17) - 64                     # a 128-row panel straddling q = 2^17
    ch = rd.Chain(11, alpha_max=1, row_begin=r0, row_end=r0 + 128)
    got = ch.read_rows(1)
    ch.close()
    sample = [0, 63, 64, 65, 127]
    want = _oracle_rows_a1(11, [r0 + i for i in sample])
    assert (got[sample] == want).all()
    # the peer all-gather chain's own panel of A^1 (RP slot) for the rank holding rows >= 2^17
    bounds = [min(N, b) for b in range(0, N + 12032, 12032)]
    if bounds[-1] != N:
        bounds.append(N)
    rank = next(s for s in range(len(bounds) - 1) if bounds[s] <= 140000 < bounds[s + 1])
    ag = rd.AgChain(11, bounds, rank, alpha_max=1)
    rows = ag.read_rows(1)
    ag.close()
    pick = [140000 - bounds[rank], bounds[rank + 1] - 1 - bounds[rank]]
    assert (rows[pick] == _oracle_rows_a1(11, [bounds[rank] + i for i in pick])).all()


@pytest.mark.parametrize("m", [1, 3, 5, 7, 8])
def test_roman_cylinder_ex_dense_equals_structured_and_formulas(m):
    """rd_roman_cylinder_ex: the dense GEMM chain (method 0) and the structured chain (method 1)
    give the same gamma; both equal the oracle chain's (Alg 1 / Prop 8) for n = 3..60."""
    ref = O.power_chain(m, 50, 10, 0) if m <= 7 else None
    for n in range(3, 61):
        g0 = rd.rd_roman_cylinder(m, n, method=0)
        g1 = rd.rd_roman_cylinder(m, n, method=1)
        assert g0 == g1, (m, n)
        if ref is not None:
            assert g0 == O.gamma_from_chain(ref, n), (m, n)
        elif m == 8:
            c = (18 * n + 4) // 5
            f8 = c if n % 5 == 0 else (c + 1 if (n % 5 in (2, 3, 4) or n == 6) else c + 2)
            assert g0 == (13 if n == 3 else f8), n     # P:443-448 with the R10 erratum at n = 3
    with pytest.raises(rd.RDError) as e:
        rd.rd_roman_cylinder(m, 5, method=2)
    assert e.value.status == rd.RD_EINVAL


# ------------------------------------------- small orders: device-resident chain --
@pytest.mark.parametrize("m", [1, 2, 3, 4, 5, 6])
def test_small_chain_kernel_equals_host_chain_and_oracle(m):
    """The device-resident Algorithm 2 (rd_set_small_chain(1), one cooperative kernel with the
    decision on the device) equals the host-driven chain and the oracle: triple,
    k_stop and every diag, under both search policies (R6), several alpha_max, and a
    kmax too small to detect (RD_NOTFOUND)."""
    for policy in (0, 1):
        for am in (5, 10):
            ref = O.power_chain(m, 50, am, policy)
            got = {}
            for small in (True, False):
                rd.rd_set_small_chain(small)
                try:
                    got[small] = rd.rd_power_sequence(m, 50, am, policy)
                finally:
                    rd.rd_set_small_chain(True)
            for g in got.values():
                assert (g["found"], g["n0"], g["alpha"], g["beta"], g["k_stop"]) == (
                    ref["found"], ref["n0"], ref["alpha"], ref["beta"], ref["k_stop"]), (m, policy, am)
                assert g["diag"][1:ref["k_stop"] + 1] == ref["diag"][1:ref["k_stop"] + 1]
    kmax = 6
    ref = O.power_chain(m, kmax, 10, 0)
    g = rd.rd_power_sequence(m, kmax, 10, 0)
    assert g["found"] == ref["found"] and g["k_stop"] == ref["k_stop"]
    assert g["diag"][1:kmax + 1] == ref["diag"][1:kmax + 1]
    if not ref["found"]:
        assert g["status"] == rd.RD_NOTFOUND


@pytest.mark.parametrize("N,seed", [(1, 1), (7, 2), (64, 3), (65, 4), (500, 5), (1024, 6)])
def test_small_chain_kernel_generic_matrices(N, seed):
    """Caller matrices up to N = 1024 through the device-resident chain (rd_power_sequence_matrix,
    method 0) equal the oracle's Algorithm 2 on the same matrix, including tile-ragged N."""
    A16 = sparse_like(N, 6, seed=seed)
    A32 = to_inf(A16, RINF, OINF, np.int32)
    ref = O.power_chain_matrix(A32, 30, 6, 0)
    got = rd.rd_power_sequence_matrix(A16, 30, 6, 0, 0)
    assert (got["found"], got["n0"], got["alpha"], got["beta"], got["k_stop"]) == (
        ref["found"], ref["n0"], ref["alpha"], ref["beta"], ref["k_stop"])
    assert got["diag"][1:ref["k_stop"] + 1] == ref["diag"][1:ref["k_stop"] + 1]


@pytest.mark.parametrize("variant", [0, 2, 3, 4, 8])
def test_tile64_chain_equals_oracle(variant):
    """128 x 64 tiles (rd_set_gemm_tile(64): 8 x 4 accumulators per thread, 3 CTAs per SM): every
    power of m = 5 and a ragged m = 7 row panel equal the oracle, for every instruction mix, with
    and without split-K."""
    rd.rd_set_gemm_tile(64)
    rd.rd_set_gemm_variant(variant)
    try:
        for m, r0, r1, split in ((5, 0, 287, True), (7, 128, 1000, True), (7, 0, 2507, False)):
            rd.rd_set_split_k(split)
            ch = rd.Chain(m, alpha_max=6, row_begin=r0, row_end=r1)
            P = {k: X for k, X in O.powers(m, 6)}
            for k in range(2, 7):
                s = ch.step().cpu().numpy()
                assert (ch.read_rows(k) == to_inf(P[k][r0:r1], OINF, RINF, np.int16)).all(), (m, k)
                assert s[0] == min(int(min(P[k][i, i] for i in range(r0, r1))), RINF)
            ch.close()
    finally:
        rd.rd_set_gemm_tile(0)
        rd.rd_set_gemm_variant(-1)
        rd.rd_set_split_k(True)


@pytest.mark.parametrize("tn", [128, 64])
def test_forced_split_k_fixup_equals_oracle(tn):
    """Split-K with the in-kernel fixup (the last CTA of a tile folds the partials and runs the
    fused epilogue): forced 2, 3, 5 and 8 ways, both tile widths, every power and stats vector
    equal the single-pass step, and the powers equal the oracle."""
    rd.rd_set_gemm_tile(tn)
    try:
        for m, r0, r1 in ((5, 0, 287), (7, 128, 1000)):
            P = {k: X for k, X in O.powers(m, 7)}
            ref = None
            for n in (0, 2, 3, 5, 8):
                rd.rd_set_split_k(n)
                ch = rd.Chain(m, alpha_max=6, row_begin=r0, row_end=r1)
                st = [ch.step().cpu().numpy() for _ in range(6)]
                rows = ch.read_rows(7)
                ch.close()
                assert (rows == to_inf(P[7][r0:r1], OINF, RINF, np.int16)).all(), (m, n)
                if ref is None:
                    ref = st
                for a, b in zip(st, ref):
                    assert (a == b).all(), (m, n)
    finally:
        rd.rd_set_split_k(1)
        rd.rd_set_gemm_tile(0)


def test_chain_tunes_dpx_mix_bit_exact():
    """Every power of a chain stays equal to the oracle's whatever DPX mix it runs with (m = 7
    on the TMA mainloop: its steps are too short for the d = 3 / 4 tuning, so the default 3),
    and an explicit variant is what the chain reports."""
    rd.rd_set_gemm_tma(2)
    try:
        P = {k: X for k, X in O.powers(7, 7)}
        ch = rd.Chain(7, alpha_max=4)
        for k in range(2, 8):
            ch.step()
            assert (ch.read_rows(k) == to_inf(P[k], OINF, RINF, np.int16)).all(), k
        assert ch.gemm_variant in (3, 4)
        ch.close()
        rd.rd_set_gemm_variant(8)
        ch = rd.Chain(7, alpha_max=4)
        for _ in range(4):
            ch.step()
        assert ch.gemm_variant == 8
        ch.close()
    finally:
        rd.rd_set_gemm_variant(-1)
        rd.rd_set_gemm_tma(1)


def test_long_cp_async_steps_tune_dpx_mix_bit_exact():
    """Long dense steps on the cp.async mainloop tune the DPX mix too (an 8-rank m = 8 row panel:
    464 tiles x 116 k-stages, tail-split by the wave model; A^4..A^11 timed as two d = 3, 4, 4, 3
    brackets, the choice used from A^12 on): sampled rows of every power equal the oracle's row
    chain (row i of A^k = row i of A^{k-1} (x) A) and the choice is 3 or 4."""
    m, r0, r1 = 8, 0, 1024
    A = O.matrix(m)
    rows = np.sort(sample_rows(r1 - r0, 16, seed=97)) + r0
    X = A[rows]
    ch = rd.Chain(m, alpha_max=4, row_begin=r0, row_end=r1)
    for k in range(2, 14):
        ch.step()
        X = O.minplus(X, A, skip=True)
        assert (ch.read_rows(k)[rows - r0] == to_inf(X, OINF, RINF, np.int16)).all(), k
    assert ch.gemm_variant in (3, 4)
    ch.close()
