"""B200-native (min,+) power pipeline for the Roman domination number of cylinders
P_m [] C_n (arXiv 2409.17658).

Thin Python binding over the C-ABI of ``librd.so`` (include/rd.h): argument marshalling
only.  Every step of the path runs in the library's kernels; PyTorch supplies device
memory, streams and (in ``dist``) process groups.  There is no CPU fallback: if the
library is missing, importing the ops raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RD_LIB", os.path.join(PKG, "librd.so"))   # RD_LIB: A/B builds (tools/)

RD_INF = 0x3FFF
RD_STAT_NONE = 2**31 - 1
RD_OK, RD_NOTFOUND, RD_EINVAL, RD_ENOMEM, RD_ECUDA, RD_ERANGE = 0, 1, -1, -2, -3, -4


class RDError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"rd status {status}: {msg}")
        self.status = status


class _Formula(ctypes.Structure):
    _fields_ = [("n0", ctypes.c_int32), ("alpha", ctypes.c_int32), ("beta", ctypes.c_int32),
                ("n_valid", ctypes.c_int32), ("C", ctypes.c_int32 * 32), ("d", ctypes.c_int32 * 32)]


class _Period(ctypes.Structure):
    _fields_ = [("found", ctypes.c_int32), ("n0", ctypes.c_int32), ("alpha", ctypes.c_int32),
                ("beta", ctypes.c_int32), ("k_stop", ctypes.c_int32)]


_lib = None


def lib():
    """Loads librd.so (raises if it has not been built: no fallback exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing; build it with `python -m paper_2409_17658_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        i64, i32, p, ci = ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int
        L.rd_last_error.restype = ctypes.c_char_p
        L.rd_set_device.argtypes = [ci]
        L.rd_build_states.argtypes = [ci, p, p]
        L.rd_build_matrix.argtypes = [ci, p, p]
        L.rd_minplus_mul.argtypes = [p, p, p, i64]
        L.rd_minplus_mul_ex.argtypes = [p, i64, p, i64, p, i64, i64, i64, i64, p]
        L.rd_minplus_mul_acc.argtypes = [p, i64, p, i64, p, i64, i64, i64, i64, p]
        L.rd_panel_stats.argtypes = [p, p, ci, i64, i64, i64, i64, ci, p, p]
        L.rd_power_sequence.argtypes = [ci, ci, p, p]
        L.rd_power_sequence_ex.argtypes = [ci, ci, ci, ci, p, p]
        L.rd_roman_cylinder.argtypes = [ci, i64, p]
        L.rd_roman_cylinder_ex.argtypes = [ci, i64, ci, p]
        L.rd_chain_create.argtypes = [ci, ci, i64, i64, p, p]
        L.rd_chain_create_ex.argtypes = [ci, ci, i64, i64, ci, p, p]
        L.rd_chain_terms_per_step.argtypes = [p]; L.rd_chain_terms_per_step.restype = ctypes.c_double
        L.rd_power_sequence_ex2.argtypes = [ci, ci, ci, ci, ci, p, p]
        L.rd_power_sequence_timed.argtypes = [ci, ci, ci, ci, ci, p, p, p]
        L.rd_power_sequence_timed.restype = ci
        L.rd_power_sequence_matrix.argtypes = [p, i64, ci, ci, ci, ci, p, p]
        L.rd_build_matrix_border.argtypes = [p, p]
        L.rd_chain_create_matrix.argtypes = [p, i64, ci, i64, i64, ci, p, p]
        L.rd_closed_form_from.argtypes = [p, p, p, p]
        L.rd_closed_form.argtypes = [ci, p, p]
        L.rd_chain_packed_operand.argtypes = [p, p, p]
        L.rd_chain_create_packed.argtypes = [ci, ci, i64, i64, p, ctypes.c_int32, p, p]
        L.rd_chain_destroy.argtypes = [p]
        L.rd_chain_order.argtypes = [p]; L.rd_chain_order.restype = i64
        L.rd_chain_current_k.argtypes = [p]
        L.rd_chain_diag1.argtypes = [p]; L.rd_chain_diag1.restype = i32
        L.rd_chain_gemm_variant.argtypes = [p]; L.rd_chain_gemm_variant.restype = ci
        L.rd_stats_len.argtypes = [ci]
        L.rd_chain_step.argtypes = [p, p]
        L.rd_chain_read_rows.argtypes = [p, ci, p]
        L.rd_stats_decide.argtypes = [p, ci, ci, ci, p, p]
        L.rd_alu_probe.argtypes = [p]
        L.rd_set_gemm_variant.argtypes = [ci]
        L.rd_set_sparse_variant.argtypes = [ci]
        L.rd_set_split_k.argtypes = [ci]
        L.rd_set_stream_k.argtypes = [ci]
        L.rd_set_gemm_tile.argtypes = [ci]
        L.rd_dense_step_plan.argtypes = [i64, i64, ci, p, p, p, p]
        L.rd_dense_step_plan.restype = ci
        L.rd_set_gemm_tile.restype = ci
        L.rd_set_small_chain.argtypes = [ci]
        L.rd_set_small_chain.restype = ci
        L.rd_set_stream_k.restype = ci
        L.rd_set_split_tail.argtypes = [ci]
        L.rd_set_split_tail.restype = ci
        L.rd_set_gemm_tma.argtypes = [ci]
        L.rd_set_gemm_tma.restype = ci
        L.rd_set_sparse_bytes.argtypes = [ci]
        L.rd_minplus_mul32.argtypes = [p, p, p, i64]
        L.rd_minplus_mul32_ex.argtypes = [p, i64, p, i64, p, i64, i64, i64, i64, p]
        L.rd_minplus_mul32.restype = ci
        L.rd_minplus_mul32_ex.restype = ci
        L.rd_agchain_create.argtypes = [ci, ci, p, ci, ci, p, p]
        L.rd_agchain_destroy.argtypes = [p]
        L.rd_agchain_ipc_handle.argtypes = [p, p, p]
        L.rd_agchain_set_peer.argtypes = [p, ci, p, p, i64]
        L.rd_agchain_ring.argtypes = [p, p, p]
        L.rd_agchain_step.argtypes = [p, p]
        L.rd_agchain_read_rows.argtypes = [p, ci, p]
        L.rd_agchain_diag1.argtypes = [p]; L.rd_agchain_diag1.restype = i32
        L.rd_agchain_order.argtypes = [p]; L.rd_agchain_order.restype = i64
        for f in ("rd_agchain_create", "rd_agchain_destroy", "rd_agchain_ipc_handle", "rd_agchain_set_peer", "rd_agchain_ring",
                  "rd_agchain_step", "rd_agchain_read_rows"):
            getattr(L, f).restype = ci
        for f in ("rd_set_device", "rd_build_states", "rd_build_matrix", "rd_minplus_mul", "rd_minplus_mul_ex",
                  "rd_power_sequence", "rd_power_sequence_ex", "rd_roman_cylinder", "rd_roman_cylinder_ex", "rd_chain_create",
                  "rd_chain_destroy", "rd_chain_current_k", "rd_stats_len", "rd_chain_step",
                  "rd_chain_read_rows", "rd_stats_decide", "rd_alu_probe", "rd_set_gemm_variant",
                  "rd_minplus_mul_acc", "rd_panel_stats", "rd_chain_create_ex", "rd_power_sequence_ex2", "rd_set_sparse_variant",
                  "rd_power_sequence_matrix", "rd_build_matrix_border", "rd_chain_create_matrix",
                  "rd_closed_form_from", "rd_closed_form", "rd_chain_packed_operand", "rd_chain_create_packed",
                  "rd_set_split_k", "rd_set_sparse_bytes"):
            getattr(L, f).restype = ci
        _lib = L
    return _lib


def _check(rc: int, allow=(RD_OK,)) -> int:
    if rc not in allow:
        raise RDError(rc, lib().rd_last_error().decode())
    return rc


def _np_ptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.c_void_p)


def _sync_device():
    """Selects torch's current CUDA device in the library's runtime (marshalling)."""
    import torch
    _check(lib().rd_set_device(torch.cuda.current_device()))


def _stream_ptr(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


# ------------------------------------------------------------------ host-side
def rd_build_states(m: int):
    """(N, words): the correct words of length m (Def 4), lexicographic a<b<c<d."""
    n = ctypes.c_int64()
    _check(lib().rd_build_states(m, None, ctypes.byref(n)))
    buf = ctypes.create_string_buffer(n.value * m)
    _check(lib().rd_build_states(m, ctypes.cast(buf, ctypes.c_void_p), ctypes.byref(n)))
    raw = buf.raw.decode()
    return n.value, [raw[i * m:(i + 1) * m] for i in range(n.value)]


def rd_build_matrix(m: int) -> np.ndarray:
    """A(G) as int16 N x N (RD_INF off the arcs)."""
    n = ctypes.c_int64()
    _check(lib().rd_build_matrix(m, None, ctypes.byref(n)))
    A = np.empty((n.value, n.value), dtype=np.int16)
    _check(lib().rd_build_matrix(m, _np_ptr(A), ctypes.byref(n)))
    return A


def rd_build_matrix_border() -> np.ndarray:
    """The App. A border / loss matrix (97 x 97 int16, RD_INF off the arcs)."""
    n = ctypes.c_int64()
    _check(lib().rd_build_matrix_border(None, ctypes.byref(n)))
    A = np.empty((n.value, n.value), dtype=np.int16)
    _check(lib().rd_build_matrix_border(_np_ptr(A), ctypes.byref(n)))
    return A


def rd_stats_decide(stats, alpha_max: int, k: int, only_alpha: int = 0):
    """(alpha, beta) if the reduced stats of power k show A^k = beta (x) A^{k-alpha}, else None."""
    s = np.ascontiguousarray(np.asarray(stats, dtype=np.int32))
    a, b = ctypes.c_int32(), ctypes.c_int32()
    ok = lib().rd_stats_decide(_np_ptr(s), alpha_max, k, only_alpha, ctypes.byref(a), ctypes.byref(b))
    return (a.value, b.value) if ok else None


def _formula_dict(f, small):
    a = f.alpha
    out = dict(n0=f.n0, alpha=a, beta=f.beta, n_valid=f.n_valid, C=[f.C[r] for r in range(a)],
               d=[f.d[r] for r in range(a)], small={n: int(small[n - 3]) for n in range(3, f.n_valid)})
    terms = []
    for r in range(a):
        terms.append(f"ceil({f.beta}n/{a}){'+' if f.d[r] >= 0 else '-'}{abs(f.d[r])} if n = {r} mod {a}")
    out["text"] = "; ".join(terms) + f"  (n >= {f.n_valid})" + (
        "; " + ", ".join(f"gamma({n}) = {v}" for n, v in out["small"].items()) if out["small"] else "")
    return out


def rd_closed_form_from(res: dict):
    """NEXT-4 on a chain result dict (found, n0, alpha, beta, k_stop, diag): per-residue
    formula gamma(n) = (beta n + C_r)/alpha = ceil(beta n/alpha) + d_r for n >= n_valid."""
    per = _Period(int(res["found"]), res["n0"], res["alpha"], res["beta"], res["k_stop"])
    diag = np.ascontiguousarray(np.asarray(res["diag"], dtype=np.int64).clip(max=2**31 - 1).astype(np.int32))
    f = _Formula()
    small = (ctypes.c_int32 * 64)()
    _check(lib().rd_closed_form_from(ctypes.byref(per), _np_ptr(diag), ctypes.byref(f), small))
    return _formula_dict(f, small)


def rd_closed_form(m: int):
    """NEXT-4 for P_m [] C_n (computes or reuses the chain on the GPU)."""
    _sync_device()
    f = _Formula()
    small = (ctypes.c_int32 * 64)()
    _check(lib().rd_closed_form(m, ctypes.byref(f), small))
    return _formula_dict(f, small)


def rd_stats_len(alpha_max: int) -> int:
    return lib().rd_stats_len(alpha_max)


# ------------------------------------------------------------------ device-side
def rd_minplus_mul(A, B, C=None):
    """C = A (x) B for square int16 CUDA tensors (row-major), on torch's current stream."""
    import torch
    assert A.is_cuda and A.dtype == torch.int16 and A.is_contiguous() and A.dim() == 2
    M, K = A.shape
    K2, N = B.shape
    assert K == K2 and B.dtype == torch.int16 and B.is_contiguous() and B.device == A.device
    if C is None:
        C = torch.empty((M, N), dtype=torch.int16, device=A.device)
    _sync_device()
    _check(lib().rd_minplus_mul_ex(A.data_ptr(), K, B.data_ptr(), N, C.data_ptr(), N, M, N, K,
                                   _stream_ptr(None)))
    return C


RD_INF32 = 0x3FFFFFFF


def rd_minplus_mul32(A, B, C=None, stream=None):
    """C = A (x) B for int32 CUDA tensors (row-major, A: M x K, B: K x N) beyond the int16
    headroom; RD_INF32 = 0x3FFFFFFF is +inf (rd.h rd_minplus_mul32_ex)."""
    import torch
    assert A.is_cuda and A.dtype == torch.int32 and A.is_contiguous() and A.dim() == 2
    M, K = A.shape
    K2, N = B.shape
    assert K == K2 and B.dtype == torch.int32 and B.is_contiguous() and B.device == A.device
    if C is None:
        C = torch.empty((M, N), dtype=torch.int32, device=A.device)
    _sync_device()
    _check(lib().rd_minplus_mul32_ex(A.data_ptr(), K, B.data_ptr(), N, C.data_ptr(), N, M, N, K,
                                     _stream_ptr(stream)))
    return C


def rd_minplus_mul_raw(A_ptr: int, B_ptr: int, C_ptr: int, N: int):
    """The literal rd_minplus_mul(A, B, C, N) (device pointers, legacy default stream)."""
    _sync_device()
    _check(lib().rd_minplus_mul(A_ptr, B_ptr, C_ptr, N))


def rd_minplus_mul_ex(A, lda, B, ldb, C, ldc, M, N, K, stream=None):
    """Strided/rectangular form on torch tensors' data pointers."""
    _sync_device()
    _check(lib().rd_minplus_mul_ex(A.data_ptr(), lda, B.data_ptr(), ldb, C.data_ptr(), ldc, M, N, K,
                                   _stream_ptr(stream)))
    return C


def rd_minplus_mul_acc(A, lda, B, ldb, C, ldc, M, N, K, stream=None, a_offset=0, b_offset=0):
    """C = min(C, A (x) B) on int16 CUDA tensors (offsets in elements into A / B)."""
    _sync_device()
    _check(lib().rd_minplus_mul_acc(A.data_ptr() + 2 * a_offset, lda, B.data_ptr() + 2 * b_offset, ldb,
                                    C.data_ptr(), ldc, M, N, K, _stream_ptr(stream)))
    return C


def rd_panel_stats(cur, prevs, diag_row0: int, alpha_max: int, stats, stream=None):
    """Stats vector (rd_chain_step layout) of row-major int16 panel `cur` against `prevs`
    (list of same-shape CUDA tensors, A^{k-1}, A^{k-2}, ...), written into `stats`."""
    _sync_device()
    rows, cols = cur.shape
    arr = (ctypes.c_void_p * max(1, len(prevs)))(*[t.data_ptr() for t in prevs])
    _check(lib().rd_panel_stats(cur.data_ptr(), arr, len(prevs), rows, cols, cur.stride(0), diag_row0,
                                alpha_max, stats.data_ptr(), _stream_ptr(stream)))
    return stats


def rd_power_sequence(m: int, kmax: int = 50, alpha_max: int = 10, policy: int = 0, method: int = 0):
    """Algorithm 2 on the GPU: dict(found, n0, alpha, beta, k_stop, diag).
    method 0: dense (min,+) GEMM steps; 1: structured steps (finite terms only, NEXT-3)."""
    _sync_device()
    out = _Period()
    diag = np.zeros(kmax + 1, dtype=np.int32)
    sec = (ctypes.c_double * 2)()
    rc = _check(lib().rd_power_sequence_timed(m, kmax, alpha_max, policy, method, ctypes.byref(out),
                                              _np_ptr(diag), sec), allow=(RD_OK, RD_NOTFOUND))
    return dict(found=bool(out.found), n0=out.n0, alpha=out.alpha, beta=out.beta, k_stop=out.k_stop,
                diag=[int(x) for x in diag], status=rc, t_build=sec[0], t_chain=sec[1])


def rd_power_sequence_matrix(A: np.ndarray, kmax: int = 50, alpha_max: int = 10, policy: int = 0,
                             method: int = 0):
    """Algorithm 2 on a caller-supplied host int16 matrix (RD_INF = inf)."""
    _sync_device()
    A = np.ascontiguousarray(A, dtype=np.int16)
    out = _Period()
    diag = np.zeros(kmax + 1, dtype=np.int32)
    rc = _check(lib().rd_power_sequence_matrix(_np_ptr(A), A.shape[0], kmax, alpha_max, policy, method,
                                               ctypes.byref(out), _np_ptr(diag)), allow=(RD_OK, RD_NOTFOUND))
    return dict(found=bool(out.found), n0=out.n0, alpha=out.alpha, beta=out.beta, k_stop=out.k_stop,
                diag=[int(x) for x in diag], status=rc)


def rd_roman_cylinder(m: int, n: int, method: int | None = None) -> int:
    """gamma_R(P_m [] C_n); method None = the library default (structured), 0 = dense GEMM
    chain, 1 = structured step (rd_roman_cylinder_ex)."""
    _sync_device()
    g = ctypes.c_int64()
    if method is None:
        _check(lib().rd_roman_cylinder(m, n, ctypes.byref(g)))
    else:
        _check(lib().rd_roman_cylinder_ex(m, n, method, ctypes.byref(g)))
    return g.value


def rd_set_gemm_variant(dpx_cols: int):
    """Mainloop instruction mix (rd.h): dpx_cols in {0, 2, 3, 4, 8}; -1 = default (3, tuned
    against 4 per long chain)."""
    _check(lib().rd_set_gemm_variant(dpx_cols))


def rd_set_gemm_tma(mode):
    """Mainloop loads of dense chain steps (rd.h rd_set_gemm_tma): 0 cp.async, 1 auto (default:
    TMA for long single-pass steps), 2 TMA always; True = 2, False = 0."""
    if isinstance(mode, bool):
        mode = 2 if mode else 0
    _check(lib().rd_set_gemm_tma(int(mode)))


def rd_set_split_k(enable):
    """Split-K policy of dense chain steps (rd.h): True/1 model (default), False/0 never,
    n >= 2 always n ways; identical results."""
    _check(lib().rd_set_split_k(int(enable) if not isinstance(enable, bool) else (1 if enable else 0)))


def rd_set_stream_k(mode: int):
    """Stream-K dense chain steps (rd.h): 0 off (default), 1 model, 2 hybrid, 3 full."""
    _check(lib().rd_set_stream_k(int(mode)))


def rd_dense_step_plan(rows: int, N: int, sms: int = 148):
    """(tile width, split count, tail-only split, predicted cost) of a dense chain step's wave
    model (rd.h)."""
    tile, ns, tail, cost = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_double()
    _check(lib().rd_dense_step_plan(rows, N, sms, ctypes.byref(tile), ctypes.byref(ns), ctypes.byref(tail),
                                    ctypes.byref(cost)))
    return tile.value, ns.value, bool(tail.value), cost.value


def rd_set_split_tail(mode: int):
    """Split form of dense chain steps (rd.h): 0 uniform, 1 wave model (default), 2 tail only."""
    _check(lib().rd_set_split_tail(int(mode)))


def rd_set_gemm_tile(tn: int):
    """Tile width of dense chain steps (rd.h): 0 = wave model (default), 64 or 128 forced."""
    _check(lib().rd_set_gemm_tile(int(tn)))


def rd_set_small_chain(enable: bool):
    """Small orders' dense Algorithm 2 as one device-resident kernel (rd.h; default on)."""
    _check(lib().rd_set_small_chain(1 if enable else 0))


def rd_set_sparse_bytes(mode):
    """Structured-step kernel for later chains: 2 slab byte kernel (default, also True),
    1 byte kernel in natural order, 0 (False) 16-bit kernel only.  Identical results."""
    if isinstance(mode, bool):
        mode = 2 if mode else 0
    _check(lib().rd_set_sparse_bytes(int(mode)))


def rd_set_sparse_variant(v: int):
    """Structured-step kernel shape (rd.h): 0..3."""
    _check(lib().rd_set_sparse_variant(v))


def rd_alu_probe():
    """Measured integer issue rates on the current device (see rd.h)."""
    _sync_device()
    out = (ctypes.c_double * 4)()
    _check(lib().rd_alu_probe(out))
    return dict(dpx_warp_instr_per_clk_sm=out[0], dpx_minplus_per_clk_sm=out[1],
                mixed_minplus_per_clk_sm=out[2], sm_mhz=out[3])


class Chain:
    """Rows [row_begin, row_end) of every power A^k of A(G) on the current device
    (rd_chain_*).  step() enqueues A^{k+1} = A^k (x) A with the fused stats."""

    def __init__(self, m: int, alpha_max: int = 10, row_begin: int = 0, row_end: int | None = None,
                 stream=None, method: int = 0, matrix: np.ndarray | None = None, packed=None,
                 diag1: int | None = None):
        import torch
        _sync_device()
        self.m, self.alpha_max = m, alpha_max
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        if row_end is None:
            row_end = count_words(m) if matrix is None else matrix.shape[0]
        self.row_begin, self.row_end = row_begin, row_end
        h = ctypes.c_void_p()
        if packed is not None:
            # dense chain over a packed operand (a torch int32/uint32 device tensor), e.g. broadcast
            _check(lib().rd_chain_create_packed(m, alpha_max, row_begin, row_end, packed.data_ptr(),
                                                2**31 - 1 if diag1 is None else diag1,
                                                _stream_ptr(self.stream), ctypes.byref(h)))
        elif matrix is None:
            _check(lib().rd_chain_create_ex(m, alpha_max, row_begin, row_end, method, _stream_ptr(self.stream),
                                            ctypes.byref(h)))
        else:
            Am = np.ascontiguousarray(matrix, dtype=np.int16)
            _check(lib().rd_chain_create_matrix(_np_ptr(Am), Am.shape[0], alpha_max, row_begin, row_end, method,
                                                _stream_ptr(self.stream), ctypes.byref(h)))
        self.method = method
        self._h = h
        self.N = lib().rd_chain_order(h)
        self.stats = torch.empty(rd_stats_len(alpha_max), dtype=torch.int32, device="cuda")

    def packed_operand(self):
        """The packed right operand as a torch int32 CUDA tensor VIEW (no copy, owned by the chain)."""
        import torch
        ptr, words = ctypes.c_void_p(), ctypes.c_int64()
        _check(lib().rd_chain_packed_operand(self._h, ctypes.byref(ptr), ctypes.byref(words)))
        return _wrap_device(ptr.value, words.value, torch.int32)

    @property
    def terms_per_step(self) -> float:
        """(min,+) terms one step evaluates (rows*N*N dense, rows*nnz(A) structured)."""
        return lib().rd_chain_terms_per_step(self._h)

    @property
    def diag1(self) -> int:
        """min over this panel's rows of A_pp (INT32_MAX if none)."""
        return lib().rd_chain_diag1(self._h)

    @property
    def k(self) -> int:
        return lib().rd_chain_current_k(self._h)

    @property
    def gemm_variant(self) -> int:
        """DPX column count of this chain's dense steps (rd_chain_gemm_variant)."""
        return lib().rd_chain_gemm_variant(self._h)

    def step(self, stats=None):
        s = self.stats if stats is None else stats
        _check(lib().rd_chain_step(self._h, ctypes.c_void_p(s.data_ptr())))
        return s

    def read_rows(self, k: int) -> np.ndarray:
        out = np.empty((self.row_end - self.row_begin, self.N), dtype=np.int16)
        _check(lib().rd_chain_read_rows(self._h, k, _np_ptr(out)))
        return out

    def close(self):
        if getattr(self, "_h", None):
            lib().rd_chain_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


RD_IPC_HANDLE_BYTES = 64


class AgChain:
    """Rows [bounds[rank], bounds[rank+1]) of every power of A(G) in the peer all-gather form
    (rd_agchain_*): A^{k+1} = A (x) A^k with A^k read from every rank's ring inside the GEMM.
    Register the other ranks with set_peer (IPC handle from another process, or a device
    pointer of this process) before the first step."""

    def __init__(self, m: int, bounds, rank: int, alpha_max: int = 10, stream=None):
        import torch
        _sync_device()
        self.m, self.alpha_max, self.rank = m, alpha_max, rank
        self.bounds = [int(b) for b in bounds]
        self.world = len(self.bounds) - 1
        self.row_begin, self.row_end = self.bounds[rank], self.bounds[rank + 1]
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        b = np.ascontiguousarray(self.bounds, dtype=np.int64)
        h = ctypes.c_void_p()
        _check(lib().rd_agchain_create(m, alpha_max, _np_ptr(b), self.world, rank, _stream_ptr(self.stream),
                                       ctypes.byref(h)))
        self._h = h
        self.N = lib().rd_agchain_order(h)
        self.stats = torch.empty(rd_stats_len(alpha_max), dtype=torch.int32, device="cuda")

    def ipc_handle(self):
        """(handle bytes, slot words) of this rank's ring, to send to the peers."""
        buf = ctypes.create_string_buffer(RD_IPC_HANDLE_BYTES)
        words = ctypes.c_int64()
        _check(lib().rd_agchain_ipc_handle(self._h, ctypes.cast(buf, ctypes.c_void_p), ctypes.byref(words)))
        return buf.raw, words.value

    def ring(self):
        """(device pointer, slot words) of this rank's ring, for peers in the same process."""
        ptr, words = ctypes.c_void_p(), ctypes.c_int64()
        _check(lib().rd_agchain_ring(self._h, ctypes.byref(ptr), ctypes.byref(words)))
        return ptr.value, words.value

    def set_peer(self, s: int, handle: bytes | None = None, ring_ptr: int | None = None,
                 slot_words: int = 0):
        hb = ctypes.create_string_buffer(handle, RD_IPC_HANDLE_BYTES) if handle is not None else None
        _check(lib().rd_agchain_set_peer(self._h, s, ctypes.cast(hb, ctypes.c_void_p) if hb is not None else None,
                                         ctypes.c_void_p(ring_ptr) if ring_ptr else None, slot_words))

    @property
    def diag1(self) -> int:
        return lib().rd_agchain_diag1(self._h)

    def step(self, stats=None):
        s = self.stats if stats is None else stats
        _check(lib().rd_agchain_step(self._h, ctypes.c_void_p(s.data_ptr())))
        return s

    def read_rows(self, k: int) -> np.ndarray:
        out = np.empty((self.row_end - self.row_begin, self.N), dtype=np.int16)
        _check(lib().rd_agchain_read_rows(self._h, k, _np_ptr(out)))
        return out

    def close(self):
        if getattr(self, "_h", None):
            lib().rd_agchain_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _wrap_device(ptr: int, n: int, dtype):
    """A torch view of library-owned device memory (via __cuda_array_interface__)."""
    import torch

    class _Buf:
        __cuda_array_interface__ = {"shape": (n,), "typestr": "<i4", "data": (ptr, False), "version": 3,
                                    "strides": None}
    return torch.as_tensor(_Buf(), device="cuda")


def count_words(m: int) -> int:
    n = ctypes.c_int64()
    _check(lib().rd_build_states(m, None, ctypes.byref(n)))
    return n.value
