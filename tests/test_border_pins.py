"""NEXT-1: the border / loss variant of Appendix A, oracle pins (CPU).

The App. A matrix (97 x 97, labels 10p(a) + 5p(b) - 2nd(q,p), Algorithm 3) runs through the
same Algorithm 2.  Pins: the paper's (n0, a, b) = (30, 1, 1); two independent
computations of 2 L_a(n) = min_g 5 g - 2|D(g)| that use neither words nor nd (X6 brute force
over the 2-sets, X7 DP over the 4 rows); Lemma 10 (2 L_a(n) >= n for n >= 10)."""
import os

import numpy as np
import pytest

import oracle as O

INF = int(O.INF)


@pytest.fixture(scope="module")
def chain():
    return O.power_chain_matrix(O.border_matrix(), 50, 10, 0)


def test_border_structure(golden):
    g = golden("border_appendix_a.json")["survey_v16"]
    A = O.border_matrix()
    fin = A != INF
    assert A.shape == (g["words"], g["words"])
    assert int(fin.sum()) == g["nnz"]
    assert int(A[fin].min()) == g["label_min"] and int(A[fin].max()) == g["label_max"]
    w = O.words(4)
    for q in range(len(w)):
        for p in np.nonzero(fin[q])[0]:
            pa, pb = w[p].count("a"), w[p].count("b")
            assert A[q, p] == 10 * pa + 5 * pb - 2 * O.nd(w[q], w[p])
    # every standard arc (m = 4) is a border arc; row 4 only relaxes (q_4 = d)
    S = O.matrix(4) != INF
    assert (fin | ~S).all()


def test_nd_cases():
    # Algorithm 3 case by case
    assert O.nd("aaaa", "aaaa") == 4 + 1          # a,a in every row, +1 for p_4 = a
    assert O.nd("dddd", "aaaa") == 12 + 1
    assert O.nd("bcbc", "cccc") == 1 + 1 + 1 + 1   # (b,c) and (c,c)
    assert O.nd("cdcd", "bcbc") == 4               # (c,d) x (b,c) cross product
    assert O.nd("cccc", "dddd") == 0


def test_border_triple_p664(golden, chain):
    g = golden("border_appendix_a.json")
    assert (chain["n0"], chain["alpha"], chain["beta"]) == tuple(g["triple"])


def test_border_diag_vs_bruteforce(chain):
    for n in range(3, 7):
        assert chain["diag"][n] == O.border_bruteforce(n), n


def test_border_diag_vs_rowdp(chain):
    for n in range(3, 11):
        assert chain["diag"][n] == O.border_rowdp(n), n


def test_border_claim_and_erratum(golden, chain):
    g = golden("border_appendix_a.json")
    lo, hi = g["claimed_equal_n_range"]
    for n in range(lo, hi + 1):
        v = O.gamma_from_chain(chain, n)
        if n == g["erratum_n"]:
            assert v == g["erratum_value"]
        else:
            assert v == n, n
    for n in range(10, 301):                      # Lemma 10 through the recurrence
        assert O.gamma_from_chain(chain, n) >= n


def test_border_erratum_n11_rowdp(golden, chain):
    """P:664's "2 L_a(n) = n for 10 <= n <= 30" fails at n = 11 (R16): the border
    chain's diagonal, the golden value written by tools/make_golden.py (oracle only) and a live
    run of the independent border row DP X7 (~10 s on 8 cores) all give 12."""
    g = golden("border_n11_rowdp.json")
    assert g["n"] == 11 and g["value"] == golden("border_appendix_a.json")["erratum_value"] == 12
    assert O.gamma_from_chain(chain, 11) == g["value"]
    assert O.border_rowdp(11) == g["value"]
