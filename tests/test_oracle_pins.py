"""Pins for the oracle (CPU only).

The oracle (oracle/rd_oracle.c) is checked against things other than itself:
values the paper prints (Tables 1 and 2, the closed formulas of P:427-463 with the
two errata of DESIGN.md R10), closed forms (gamma_R(C_n) = ceil(2n/3); Cor 12 /
Remark 13), brute force by four independent routes (X1 exhaustive f, X2 S2-subset,
X3 row DP, X5 column-pair trace DP — none uses words, the matrix or the product),
semiring identities, and the survey's independent checksums (V24).
"""
import numpy as np
import pytest

import oracle as O

INF = int(O.INF)


# ------------------------------------------------------------------ Table 1 --
def test_word_counts_table1(golden):
    g = golden("table1_word_counts.json")["counts"]
    for m, c in g.items():
        assert O.count_words(int(m)) == c, m
    assert O.count_words(1) == 4


def test_words_are_lexicographic_and_correct():
    for m in range(1, 6):
        w = O.words(m)
        assert w == sorted(w)
        assert len(set(w)) == len(w)
        for x in w:
            assert all(c in "abcd" for c in x) and len(x) == m


# ------------------------------------------------ gamma vs brute force (pins) --
def _chain(m, kmax=50, alpha_max=10, policy=0):
    return O.power_chain(m, kmax, alpha_max, policy)


@pytest.fixture(scope="module")
def chains():
    return {m: _chain(m) for m in range(1, 7)}


def test_diag_equals_exhaustive_bruteforce(chains):
    # X1: every f: V -> {0,1,2} (north star: m <= 3, n <= 6)
    for m in (1, 2, 3):
        for n in range(3, 7):
            if m * n > 18:
                continue
            assert chains[m]["diag"][n] == O.gamma_bruteforce3(m, n), (m, n)


def test_diag_equals_s2_subset(chains):
    # X2: mn <= 24
    for m in range(1, 7):
        for n in range(3, 9):
            if m * n > 24:
                continue
            assert O.gamma_from_chain(chains[m], n) == O.gamma_s2subset(m, n), (m, n)


def test_diag_equals_row_dp(chains):
    # X3 along the path; covers m = 6 and n up to 8
    for m in range(1, 7):
        for n in range(3, 8):
            assert O.gamma_from_chain(chains[m], n) == O.gamma_rowdp(m, n), (m, n)


def test_diag_equals_pair_trace_config1(chains):
    # X5 along the cycle: config 1 (m = 3, n = 3..30) and m = 1, 2, 4
    for m in (1, 2, 3, 4):
        for n in range(3, 31):
            assert O.gamma_from_chain(chains[m], n) == O.gamma_pairtrace(m, n), (m, n)


def test_bruteforces_agree_with_each_other():
    for m, n in [(1, 5), (2, 4), (2, 7), (3, 4), (3, 5)]:
        x1 = O.gamma_bruteforce3(m, n)
        assert x1 == O.gamma_s2subset(m, n) == O.gamma_rowdp(m, n) == O.gamma_pairtrace(m, n), (m, n)


def test_known_small_values():
    # P_2 [] C_4 is the 3-cube Q_3: two antipodal 2s dominate it, weight 4.
    assert O.gamma_s2subset(2, 4) == 4
    assert O.gamma_bruteforce3(2, 4) == 4


# ------------------------------------------------------------ closed forms --
def test_m1_closed_form(chains):
    # gamma_R(C_n) = ceil(2n/3) (Cockayne et al.), n = 3..60 through the recurrence
    for n in range(3, 61):
        assert O.gamma_from_chain(chains[1], n) == (2 * n + 2) // 3, n


def test_remark13_and_cor12_equality(chains):
    # gamma_R = 2(m+1)n/5 for m >= 4 and 5 | n (Cor 12 P:501-507, Remark 13 P:513-514)
    for m in (4, 5, 6):
        for n in range(5, 51, 5):
            assert O.gamma_from_chain(chains[m], n) == 2 * (m + 1) * n // 5, (m, n)
    # and for m = 7, 8, 9 via the row DP at n = 5 (independent of the matrix)
    for m in (7, 8, 9):
        assert O.gamma_rowdp(m, 5) == 2 * (m + 1) * 5 // 5


def test_remark13_smaller_for_m2_m3(chains):
    # "the Roman domination number is smaller if m = 2, 3": never larger, and
    # strictly smaller somewhere along n = 5k
    for m in (2, 3):
        vals = [(O.gamma_from_chain(chains[m], n), 2 * (m + 1) * n // 5) for n in range(5, 51, 5)]
        assert all(g <= b for g, b in vals)
        assert any(g < b for g, b in vals)


# ------------------------------------------------------------- Table 2 pins --
def test_table2_periods_canonical_and_paper_compat(golden, chains):
    g = golden("table2_periods.json")
    for m in range(2, 7):
        n0, a, b = g["table2"][str(m)]
        r = chains[m]
        got = (r["n0"], r["alpha"], r["beta"])
        if m == 4:
            assert got == tuple(g["first_detection_m4"])
        else:
            assert got == (n0, a, b), m
        rc = O.power_chain(m, 50, 5, 1)
        assert (rc["n0"], rc["alpha"], rc["beta"]) == (n0, a, b), m


def test_table2_m7(golden):
    g = golden("table2_periods.json")["table2"]["7"]
    r = _chain(7, alpha_max=5)
    assert (r["n0"], r["alpha"], r["beta"]) == tuple(g)
    assert r["k_stop"] == 26


@pytest.fixture(scope="module")
def chain8():
    return _chain(8, alpha_max=5)


@pytest.mark.slow
def test_table2_m8(golden, chain8):
    g = golden("table2_periods.json")["table2"]["8"]
    r = chain8
    assert (r["n0"], r["alpha"], r["beta"]) == tuple(g)
    assert r["k_stop"] == 26


def test_lemma2_persistence():
    # Lemma 2: once A^{n0+a} = b (x) A^{n0}, it holds for every n >= n0.
    for m in (2, 3, 4, 5):
        r = _chain(m)
        n0, a, b = r["n0"], r["alpha"], r["beta"]
        P = {k: X for k, X in O.powers(m, min(50, n0 + a + 12))}
        for n in range(n0, n0 + 12):
            assert O.shift(P[n + a], P[n]) == b, (m, n)
        if n0 - 1 >= 1:
            assert O.shift(P[n0 - 1 + a], P[n0 - 1]) is None  # n0 is minimal for this alpha


# -------------------------------------------------- formulas with errata --
def _f7(n):
    c = (16 * n + 4) // 5
    return c if n % 5 == 0 else c + 1


def _f8(n):
    c = (18 * n + 4) // 5
    if n % 5 == 0:
        return c
    if n % 5 in (2, 3, 4) or n == 6:
        return c + 1
    return c + 2


def _f9(n):
    return 4 * n if n % 5 == 0 else 4 * n + 2


def test_formula_m7_with_erratum(golden):
    er = golden("formulas_m7_m8_m9.json")["errata"]["7,6"]
    r = _chain(7)
    for n in range(3, 61):
        g = O.gamma_from_chain(r, n)
        if n == 6:
            assert _f7(n) == er["formula"] and g == er["true"]
        else:
            assert g == _f7(n), n


def test_erratum_witness_7_6(golden):
    w = golden("formulas_m7_m8_m9.json")["witness_7_6"]
    f = np.array([[int(c) for c in row] for row in w], dtype=np.int32)
    assert f.shape == (7, 6)
    assert O.rdf_weight(f) == 20          # a valid RDF of weight 20 < formula 21
    assert O.gamma_rowdp(7, 6) == 20
    # the checker rejects what is not an RDF (Def): every 0 needs a neighbour with 2
    for r, c in zip(*np.nonzero(f == 2)):
        g = f.copy()
        g[r, c] = 0                        # drop one 2: some 0 (or this vertex) loses its 2-neighbour
        assert O.rdf_weight(g) == -1, (r, c)
    g = f.copy()
    g[0, 0] = 3                            # values outside {0, 1, 2}
    assert O.rdf_weight(g) == -1
    g = f.copy()
    g[g == 0] = 1                          # all-nonzero: valid, weight = sum of values
    assert O.rdf_weight(g) == int(g.sum())
    # domination wraps around the cycle (columns n-1 and 0 are adjacent) but not the path ends
    h = np.zeros((1, 4), dtype=np.int32)
    h[0, 0], h[0, 2] = 2, 0
    h[0, 2] = 2
    assert O.rdf_weight(h) == 4
    h = np.zeros((2, 3), dtype=np.int32)
    h[0, 0] = 2                            # (0,1) (0,2) via the cycle, (1,0) below; (1,1) undominated
    assert O.rdf_weight(h) == -1
    h[1, 1] = 1
    h[1, 2] = 1
    assert O.rdf_weight(h) == 4


def test_erratum_8_3():
    assert _f8(3) == 12
    assert O.gamma_s2subset(8, 3) == 13   # exhaustive over 2^24 S2 sets
    assert O.gamma_rowdp(8, 3) == 13


def test_formulas_m8_m9_small_n_rowdp():
    # independent of the matrix: X3 for n = 3..8
    for n in range(3, 9):
        want8 = 13 if n == 3 else _f8(n)
        assert O.gamma_rowdp(8, n) == want8, n
        assert O.gamma_rowdp(9, n) == _f9(n), n


@pytest.mark.slow
def test_formula_m8_full_chain(golden, chain8):
    r = chain8
    for n in range(3, 61):
        g = O.gamma_from_chain(r, n)
        assert g == (13 if n == 3 else _f8(n)), n


# ------------------------------------------------------ semiring --
def _rand(rng, r, c, inf_frac=0.2, hi=20):
    X = rng.integers(0, hi + 1, size=(r, c)).astype(np.int32)
    X[rng.random((r, c)) < inf_frac] = INF
    return X


def test_spec_worked_product():
    # hand-evaluated: C00 = min(1+0, 2+1) = 1, C11 = min(3+5, inf+0) = 8 (SPEC trop_mul example)
    A = np.array([[1, 2], [3, INF]], dtype=np.int32)
    B = np.array([[0, 5], [1, 0]], dtype=np.int32)
    assert O.minplus(A, B).tolist() == [[1, 2], [3, 8]]


def test_identity_associativity_scalar():
    rng = np.random.default_rng(0)
    for _ in range(200):
        n = int(rng.integers(1, 9))
        A, B, C = (_rand(rng, n, n) for _ in range(3))
        I = np.full((n, n), INF, dtype=np.int32)
        np.fill_diagonal(I, 0)
        assert (O.minplus(A, I) == A).all() and (O.minplus(I, A) == A).all()
        assert (O.minplus(O.minplus(A, B), C) == O.minplus(A, O.minplus(B, C))).all()
        al = int(rng.integers(0, 10))
        sB = np.where(B == INF, INF, B + al).astype(np.int32)
        AB = O.minplus(A, B)
        assert (O.minplus(A, sB) == np.where(AB == INF, INF, AB + al)).all()
        assert O.shift(np.where(AB == INF, INF, AB + al).astype(np.int32), AB) in (
            (al,) if (AB != INF).any() else (None,))


def test_minplus_bruteforce_tiny_rectangular():
    # every entry against an explicit enumeration of all k (python ints, no INF guard:
    # INF mapped to a large float)
    rng = np.random.default_rng(1)
    for _ in range(50):
        M, K, N = (int(x) for x in rng.integers(1, 7, size=3))
        A, B = _rand(rng, M, K, 0.3), _rand(rng, K, N, 0.3)
        C = O.minplus(A, B)
        for i in range(M):
            for j in range(N):
                cands = [float(A[i, k]) + float(B[k, j]) for k in range(K)
                         if A[i, k] != INF and B[k, j] != INF]
                assert C[i, j] == (int(min(cands)) if cands else INF)


def test_skip_form_equals_dense():
    rng = np.random.default_rng(2)
    for inf_frac in (0.0, 0.01, 0.5, 0.95, 1.0):
        A, B = _rand(rng, 57, 33, inf_frac, 300), _rand(rng, 33, 41, inf_frac, 300)
        assert (O.minplus(A, B) == O.minplus(A, B, skip=True)).all()
        assert (O.minplus(A, B) == O.minplus_bt(A, np.ascontiguousarray(B.T))).all()
    A = O.matrix(5)
    X = O.minplus(A, A)
    assert (O.minplus(X, A) == O.minplus(X, A, skip=True)).all()


def test_shift_semantics():
    Q = np.array([[0, 1], [2, 2]], dtype=np.int32)
    assert O.shift(np.array([[1, 2], [3, 4]], dtype=np.int32), Q) is None   # diffs 1,1,1,2
    assert O.shift(Q + 7, Q) == 7 and O.shift(Q, Q) == 0
    allinf = np.full((2, 2), INF, dtype=np.int32)
    assert O.shift(allinf, allinf) is None          # no finite entry fixes beta
    P = Q.copy(); P[0, 0] = INF
    assert O.shift(P, Q) is None                     # INF patterns differ


# --------------------------------------------------- structure / checksums --
def test_matrix_structure(golden):
    g = golden("survey_checksums_v24.json")
    for m in range(1, 8):
        A = O.matrix(m)
        fin = A != INF
        if str(m) in g["nnz_v11"]:
            assert int(fin.sum()) == g["nnz_v11"][str(m)], m
        assert int(np.diag(fin).sum()) == g["self_loops_v28"][str(m)], m
        # labels depend on p only: each column's finite entries are equal
        w = O.words(m)
        lab = np.array([O.label(p) for p in w])
        assert (A[fin] == np.broadcast_to(lab[None, :], A.shape)[fin]).all()
        # mirror symmetry of the rules (rows read bottom-up give the same digraph)
        idx = {x: i for i, x in enumerate(w)}
        rev = np.array([idx[x[::-1]] for x in w])
        assert (fin[np.ix_(rev, rev)] == fin).all()
        # no ab / ba / bb across an arc in the same row (Remark 3)
        for q in range(len(w)):
            for p in np.nonzero(fin[q])[0]:
                for x, y in zip(w[q], w[p]):
                    assert (x, y) not in (("a", "b"), ("b", "a"), ("b", "b"))


def test_v24_checksums(golden):
    g = golden("survey_checksums_v24.json")["checksums"]
    for m in range(1, 8):
        want = g[str(m)]
        for k, X in O.powers(m, max(int(x) for x in want)):
            if str(k) not in want:
                continue
            fin = X != INF
            got = [int((~fin).sum()), int(X[fin].astype(np.int64).sum()),
                   int(np.diag(X)[np.diag(fin)].astype(np.int64).sum())]
            assert got == want[str(k)], (m, k)
