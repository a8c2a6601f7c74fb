"""The parity oracle — TEST INFRASTRUCTURE ONLY.

A plain CPU implementation of what arXiv 2409.17658 computes (rd_oracle.c, C with
OpenMP over output rows) plus numpy marshalling.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl reference``
leg may import this package.  It shares no code with ``paper_2409_17658_b200``
and never imports it.

Infinity is ``INF = 2**31 - 1`` (int32) here; the product uses an int16 sentinel,
mapped to this one only inside the tests.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "rd_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")
INF = np.int32(2**31 - 1)

_lib = None


def build(force: bool = False) -> str:
    """Compile rd_oracle.c into liboracle.so with gcc (plain -O2, OpenMP over rows)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-Wall", "-o", tmp, SRC])
        os.replace(tmp, LIB)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB)
        i64, i32, p = ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p
        L.or_words.argtypes = [ctypes.c_int, p]; L.or_words.restype = i64
        L.or_can_follow.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int]; L.or_can_follow.restype = ctypes.c_int
        L.or_label.argtypes = [ctypes.c_char_p, ctypes.c_int]; L.or_label.restype = ctypes.c_int
        L.or_matrix.argtypes = [ctypes.c_int, p]; L.or_matrix.restype = i64
        L.or_minplus.argtypes = [p, p, p, i64, i64, i64]; L.or_minplus.restype = None
        L.or_minplus_bt.argtypes = [p, p, p, i64, i64, i64]; L.or_minplus_bt.restype = None
        L.or_minplus_skip.argtypes = [p, p, p, i64, i64, i64]; L.or_minplus_skip.restype = None
        L.or_diag_min.argtypes = [p, i64]; L.or_diag_min.restype = i32
        L.or_shift.argtypes = [p, p, i64, p]; L.or_shift.restype = ctypes.c_int
        L.or_power_chain.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, p, p, p]
        L.or_power_chain.restype = ctypes.c_int
        for f in ("or_gamma_bruteforce3", "or_gamma_s2subset", "or_gamma_rowdp", "or_gamma_pairtrace"):
            getattr(L, f).argtypes = [ctypes.c_int, ctypes.c_int]
            getattr(L, f).restype = i32
        L.or_rdf_weight.argtypes = [ctypes.c_int, ctypes.c_int, p]; L.or_rdf_weight.restype = i32
        L.or_power_chain_matrix.argtypes = [p, i64, ctypes.c_int, ctypes.c_int, ctypes.c_int, p, p, p]
        L.or_power_chain_matrix.restype = ctypes.c_int
        L.or_can_follow_border.argtypes = [ctypes.c_char_p, ctypes.c_char_p]; L.or_can_follow_border.restype = ctypes.c_int
        L.or_nd.argtypes = [ctypes.c_char_p, ctypes.c_char_p]; L.or_nd.restype = ctypes.c_int
        L.or_border_matrix.argtypes = [p]; L.or_border_matrix.restype = i64
        L.or_border_bruteforce.argtypes = [ctypes.c_int]; L.or_border_bruteforce.restype = i32
        L.or_border_rowdp.argtypes = [ctypes.c_int]; L.or_border_rowdp.restype = i32
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.c_void_p)


# ---------------------------------------------------------------- words/matrix
def count_words(m: int) -> int:
    """C_m, the number of correct words of length m (Def 4; Table 1)."""
    return int(lib().or_words(m, None))


def words(m: int) -> list[str]:
    """Correct words of length m in lexicographic order a<b<c<d (Def 4)."""
    n = count_words(m)
    buf = ctypes.create_string_buffer(n * m)
    lib().or_words(m, ctypes.cast(buf, ctypes.c_void_p))
    raw = buf.raw.decode()
    return [raw[i * m:(i + 1) * m] for i in range(n)]


def can_follow(q: str, p: str) -> bool:
    """p can follow q (reading R1 p_i=d)."""
    return bool(lib().or_can_follow(q.encode(), p.encode(), len(q)))


def label(p: str) -> int:
    """l(q,p) = 2 p(a) + p(b)."""
    return int(lib().or_label(p.encode(), len(p)))


def matrix(m: int) -> np.ndarray:
    """A(G): int32 N x N, INF off the arcs (Cor 7)."""
    n = count_words(m)
    A = np.empty((n, n), dtype=np.int32)
    lib().or_matrix(m, _ptr(A))
    return A


# ---------------------------------------------------------------- semiring ops
def minplus(A: np.ndarray, B: np.ndarray, skip: bool = False) -> np.ndarray:
    """C = A (x) B, c_ij = min_k(a_ik + b_kj).  int32 with INF = 2**31-1."""
    A = np.ascontiguousarray(A, dtype=np.int32)
    B = np.ascontiguousarray(B, dtype=np.int32)
    M, K = A.shape
    K2, N = B.shape
    assert K == K2
    C = np.empty((M, N), dtype=np.int32)
    (lib().or_minplus_skip if skip else lib().or_minplus)(_ptr(A), _ptr(B), _ptr(C), M, N, K)
    return C


def minplus_bt(A: np.ndarray, BT: np.ndarray) -> np.ndarray:
    """C = A (x) B given BT = B transposed (N x K): c_ij = min_k(a_ik + bt_jk)."""
    A = np.ascontiguousarray(A, dtype=np.int32)
    BT = np.ascontiguousarray(BT, dtype=np.int32)
    M, K = A.shape
    N, K2 = BT.shape
    assert K == K2
    C = np.empty((M, N), dtype=np.int32)
    lib().or_minplus_bt(_ptr(A), _ptr(BT), _ptr(C), M, N, K)
    return C


def diag_min(X: np.ndarray) -> int:
    """min_p (X)_pp (Cor 7)."""
    X = np.ascontiguousarray(X, dtype=np.int32)
    return int(lib().or_diag_min(_ptr(X), X.shape[0]))


def shift(P: np.ndarray, Q: np.ndarray):
    """beta if P = beta (x) Q for a natural beta (Lemma 2), else None."""
    P = np.ascontiguousarray(P, dtype=np.int32)
    Q = np.ascontiguousarray(Q, dtype=np.int32)
    b = np.zeros(1, dtype=np.int32)
    ok = lib().or_shift(_ptr(P), _ptr(Q), P.size, _ptr(b))
    return int(b[0]) if ok else None


def power_chain(m: int, kmax: int = 50, alpha_max: int = 10, policy: int = 0, want_final: bool = False):
    """Algorithm 2 with the first-detection search (R6).

    Returns dict(found, n0, alpha, beta, k_stop, diag[list, index k], final[A^k_stop or None]).
    """
    diag = np.zeros(kmax + 1, dtype=np.int32)
    out = np.zeros(5, dtype=np.int32)
    final = None
    fp = None
    if want_final:
        n = count_words(m)
        final = np.empty((n, n), dtype=np.int32)
        fp = _ptr(final)
    rc = lib().or_power_chain(m, kmax, alpha_max, policy, _ptr(diag), _ptr(out), fp)
    if rc != 0:
        raise ValueError("or_power_chain failed")
    return dict(found=bool(out[0]), n0=int(out[1]), alpha=int(out[2]), beta=int(out[3]),
                k_stop=int(out[4]), diag=[int(x) for x in diag], final=final)


def powers(m: int, kmax: int):
    """Yield (k, A^k) for k = 1..kmax, A^k = A^{k-1} (x) A (Alg 2 step 3)."""
    A = matrix(m)
    X = A.copy()
    yield 1, X
    for k in range(2, kmax + 1):
        X = minplus(X, A, skip=True)
        yield k, X


def gamma_from_chain(res: dict, n: int) -> int:
    """gamma_R(P_m [] C_n) from a detected (n0, alpha, beta) (Prop 8 P:237-244 and the
    finite-difference solution P:248): n' = n0 + ((n - n0) mod alpha), gamma(n) =
    diag[n'] + beta * (n - n') / alpha, for n >= n0; diag[n] directly for n < n0."""
    d = res["diag"]
    if n < len(d) and (not res["found"] or n <= res["k_stop"]):
        return d[n]
    assert res["found"] and n >= res["n0"]
    n0, a, b = res["n0"], res["alpha"], res["beta"]
    np_ = n0 + (n - n0) % a
    return d[np_] + b * (n - np_) // a


# ------------------------------------------------------------- brute forces
def gamma_bruteforce3(m: int, n: int) -> int:
    """(X1) min weight over all f: V -> {0,1,2} that are Roman dominating; mn <= 20."""
    return int(lib().or_gamma_bruteforce3(m, n))


def gamma_s2subset(m: int, n: int) -> int:
    """(X2) min over S2 of 2|S2| + |V minus N[S2]|; mn <= 30."""
    return int(lib().or_gamma_s2subset(m, n))


def gamma_rowdp(m: int, n: int) -> int:
    """(X3) row DP along the path, state = S2 masks of two rows; n <= 10."""
    return int(lib().or_gamma_rowdp(m, n))


def gamma_pairtrace(m: int, n: int) -> int:
    """(X5) trace DP along the cycle over (S2 of column j-1, S2 of column j); m <= 5."""
    return int(lib().or_gamma_pairtrace(m, n))


def rdf_weight(f) -> int:
    """Weight of f if it is a Roman dominating function of P_m [] C_n, else -1."""
    f = np.ascontiguousarray(f, dtype=np.int32)
    m, n = f.shape
    return int(lib().or_rdf_weight(m, n, _ptr(f)))


# ------------------------------------------------ border / loss variant (App. A)
def border_matrix() -> np.ndarray:
    """The App. A matrix: 97 x 97 int32, labels 10p(a)+5p(b)-2nd (Alg 3)."""
    n = int(lib().or_border_matrix(None))
    A = np.empty((n, n), dtype=np.int32)
    lib().or_border_matrix(_ptr(A))
    return A


def nd(q: str, p: str) -> int:
    """Algorithm 3: newly dominated vertices nd(q, p)."""
    return int(lib().or_nd(q.encode(), p.encode()))


def can_follow_border(q: str, p: str) -> bool:
    return bool(lib().or_can_follow_border(q.encode(), p.encode()))


def power_chain_matrix(A: np.ndarray, kmax: int = 50, alpha_max: int = 10, policy: int = 0):
    """Algorithm 2 on a given int32 matrix (INF = 2**31-1)."""
    A = np.ascontiguousarray(A, dtype=np.int32)
    diag = np.zeros(kmax + 1, dtype=np.int32)
    out = np.zeros(5, dtype=np.int32)
    rc = lib().or_power_chain_matrix(_ptr(A), A.shape[0], kmax, alpha_max, policy, _ptr(diag), _ptr(out), None)
    if rc != 0:
        raise ValueError("or_power_chain_matrix failed")
    return dict(found=bool(out[0]), n0=int(out[1]), alpha=int(out[2]), beta=int(out[3]),
                k_stop=int(out[4]), diag=[int(x) for x in diag], final=None)


def border_bruteforce(n: int) -> int:
    """(X6) 2 L_a(n) = min_g 5 g - 2|D(g)| over almost-RDFs of P_4 [] C_n."""
    return int(lib().or_border_bruteforce(n))


def border_rowdp(n: int) -> int:
    """(X7) 2 L_a(n) by a DP over the 4 rows; n <= 10."""
    return int(lib().or_border_rowdp(n))
