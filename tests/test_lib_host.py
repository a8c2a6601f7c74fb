"""librd.so on the CPU: the library loads and exports every symbol include/rd.h
declares; the host half (rd_build_states, rd_build_matrix, rd_stats_decide, argument
validation) is bit-exact against the oracle.  No GPU compute is called here."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle as O
import paper_2409_17658_b200 as rd
from rd_inputs import to_inf

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "rd.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rd_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = rd.lib()
    names = _header_functions()
    assert "rd_minplus_mul" in names and "rd_power_sequence" in names and "rd_roman_cylinder" in names
    for n in names:
        assert hasattr(L, n), n
    # and the .so really is an sm_100a build (fat binary inside)
    out = os.popen(f"cuobjdump --list-elf {rd.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out


def test_build_states_matches_oracle():
    for m in range(1, 12):
        n, _ = (rd.count_words(m), None)
        assert n == O.count_words(m), m
    for m in range(1, 9):
        n, words = rd.rd_build_states(m)
        assert words == O.words(m), m


@pytest.mark.parametrize("m", range(1, 9))
def test_build_matrix_bit_exact(m):
    A = rd.rd_build_matrix(m)
    B = to_inf(O.matrix(m), int(O.INF), rd.RD_INF, np.int16)
    assert A.shape == B.shape
    assert (A == B).all()


@pytest.mark.slow
def test_build_matrix_bit_exact_m9():
    A = rd.rd_build_matrix(9)
    B = to_inf(O.matrix(9), int(O.INF), rd.RD_INF, np.int16)
    assert (A == B).all()


def test_stats_decide_logic():
    am = 3
    INT_MAX = 2**31 - 1

    def stats(entries, diag=5):
        s = [diag]
        for lo, hi, mis, fin in entries:
            s += [lo, -hi, -mis, -fin]
        s += [INT_MAX, INT_MAX, 0, 0] * (am - len(entries))
        return np.array(s, dtype=np.int32)

    assert rd.rd_stats_decide(stats([(2, 2, 0, 1)]), am, 5) == (1, 2)
    assert rd.rd_stats_decide(stats([(2, 3, 0, 1), (4, 4, 0, 1)]), am, 5) == (2, 4)
    assert rd.rd_stats_decide(stats([(2, 2, 1, 1)]), am, 5) is None       # inf pattern differs
    assert rd.rd_stats_decide(stats([(INT_MAX, -INT_MAX, 0, 0)]), am, 5) is None  # nothing finite
    assert rd.rd_stats_decide(stats([(-1, -1, 0, 1)]), am, 5) is None     # beta must be natural
    # alpha is limited to k-1
    assert rd.rd_stats_decide(stats([(9, 9, 1, 1), (4, 4, 0, 1)]), am, 2) is None
    assert rd.rd_stats_decide(stats([(2, 2, 0, 1), (4, 4, 0, 1)]), am, 5, only_alpha=2) == (2, 4)


def test_argument_validation_host_paths():
    L = rd.lib()
    n = ctypes.c_int64()
    assert L.rd_build_states(0, None, ctypes.byref(n)) == rd.RD_EINVAL
    assert L.rd_build_states(3, None, None) == rd.RD_EINVAL
    assert L.rd_build_matrix(13, None, ctypes.byref(n)) == rd.RD_EINVAL
    assert b"out of range" in L.rd_last_error()
    per = rd._Period()
    # headroom: 2*m*kmax >= RD_INF is refused before any device work
    assert L.rd_power_sequence_ex(9, 1000, 10, 0, ctypes.byref(per), None) == rd.RD_ERANGE
    assert L.rd_power_sequence_ex(0, 50, 10, 0, ctypes.byref(per), None) == rd.RD_EINVAL
    assert L.rd_power_sequence_ex(3, 1, 10, 0, ctypes.byref(per), None) == rd.RD_EINVAL
    assert L.rd_power_sequence_ex(3, 50, 33, 0, ctypes.byref(per), None) == rd.RD_EINVAL
    assert L.rd_power_sequence_ex(3, 50, 10, 2, ctypes.byref(per), None) == rd.RD_EINVAL
    g = ctypes.c_int64()
    assert L.rd_roman_cylinder(3, 2, ctypes.byref(g)) == rd.RD_EINVAL
    assert L.rd_roman_cylinder(0, 5, ctypes.byref(g)) == rd.RD_EINVAL
    assert L.rd_minplus_mul(None, None, None, 4) == rd.RD_EINVAL
    assert L.rd_minplus_mul32(None, None, None, 4) == rd.RD_EINVAL
    assert L.rd_minplus_mul32_ex(None, 4, None, 4, None, 4, 0, 4, 4, None) == rd.RD_EINVAL
    b = np.array([0, 100, 287], dtype=np.int64)
    h = ctypes.c_void_p()
    assert L.rd_agchain_create(5, 10, rd._np_ptr(b), 2, 0, None, ctypes.byref(h)) == rd.RD_EINVAL  # 100 % 128
    assert L.rd_agchain_create(13, 10, rd._np_ptr(b), 2, 0, None, ctypes.byref(h)) == rd.RD_EINVAL
    assert L.rd_agchain_create(5, 10, rd._np_ptr(b), 2, 2, None, ctypes.byref(h)) == rd.RD_EINVAL  # rank
    assert L.rd_agchain_step(None, None) == rd.RD_EINVAL
    assert L.rd_chain_create_ex(12, 10, 0, 10, 0, None, ctypes.byref(h)) == rd.RD_EINVAL        # m=12 dense
    assert L.rd_set_gemm_tma(4) == rd.RD_EINVAL and L.rd_set_gemm_tma(-1) == rd.RD_EINVAL
    assert L.rd_set_gemm_tma(1) == rd.RD_OK
    assert L.rd_set_split_tail(3) == rd.RD_EINVAL and L.rd_set_split_tail(-1) == rd.RD_EINVAL
    assert L.rd_set_split_tail(1) == rd.RD_OK
    assert L.rd_set_stream_k(4) == rd.RD_EINVAL and L.rd_set_stream_k(-1) == rd.RD_EINVAL
    assert L.rd_set_stream_k(0) == rd.RD_OK
    assert L.rd_stats_len(10) == 41
    assert L.rd_set_sparse_bytes(3) == rd.RD_EINVAL and L.rd_set_sparse_bytes(-1) == rd.RD_EINVAL
    assert L.rd_set_sparse_bytes(2) == rd.RD_OK


def test_build_matrix_border_bit_exact():
    A = rd.rd_build_matrix_border()
    B = to_inf(O.border_matrix(), int(O.INF), rd.RD_INF, np.int16)
    assert A.shape == (97, 97)
    assert (A == B).all()


def test_power_sequence_matrix_argument_checks():
    L = rd.lib()
    per = rd._Period()
    A = np.full((5, 5), rd.RD_INF, dtype=np.int16)
    A[0, 1] = -3
    assert L.rd_power_sequence_matrix(rd._np_ptr(A), 5, 50, 10, 0, 0, ctypes.byref(per), None) == rd.RD_EINVAL
    A[0, 1] = 400                                   # 400 * 50 >= RD_INF: headroom
    assert L.rd_power_sequence_matrix(rd._np_ptr(A), 5, 50, 10, 0, 0, ctypes.byref(per), None) == rd.RD_ERANGE
    assert L.rd_power_sequence_matrix(None, 5, 50, 10, 0, 0, ctypes.byref(per), None) == rd.RD_EINVAL


# --------------------------------------------------------- NEXT-4 closed form
def _paper_d(m):
    # the paper's per-residue offsets over ceil(beta n / 5)
    return {7: [0, 1, 1, 1, 1], 8: [0, 2, 1, 1, 1], 9: [0, 2, 2, 2, 2]}[m]


def test_closed_form_from_oracle_chains():
    r1 = rd.rd_closed_form_from(O.power_chain(1, 50, 10, 0))
    assert (r1["alpha"], r1["beta"], r1["d"], r1["n_valid"]) == (3, 2, [0, 0, 0], 3)   # ceil(2n/3)
    r7 = rd.rd_closed_form_from(O.power_chain(7, 50, 10, 0))
    assert (r7["alpha"], r7["beta"], r7["d"]) == (5, 16, _paper_d(7))
    assert r7["n_valid"] == 7 and r7["small"][6] == 20          # erratum R10: formula gives 21
    for n in range(7, 200):
        g = (r7["beta"] * n + r7["C"][n % 5]) // 5
        assert g == -(-16 * n // 5) + (0 if n % 5 == 0 else 1)


@pytest.mark.slow
def test_closed_form_m8_oracle():
    r8 = rd.rd_closed_form_from(O.power_chain(8, 50, 10, 0))
    assert (r8["alpha"], r8["beta"], r8["d"]) == (5, 18, _paper_d(8))
    assert r8["small"] == {3: 13, 4: 16, 5: 18, 6: 23}          # n = 3 erratum, n = 6 special case


def test_closed_form_rejects_bad_input():
    with pytest.raises(rd.RDError):
        rd.rd_closed_form_from(dict(found=False, n0=0, alpha=0, beta=0, k_stop=5, diag=[0] * 6))
    bad = O.power_chain(3, 50, 10, 0)
    bad["diag"][bad["k_stop"]] += 1
    with pytest.raises(rd.RDError):
        rd.rd_closed_form_from(bad)


OOM_SCRIPT = r"""
import ctypes, resource, sys
sys.path.insert(0, sys.argv[1])
import paper_2409_17658_b200 as rd
L = rd.lib()
n = ctypes.c_int64()
assert L.rd_build_states(12, None, ctypes.byref(n)) == 0 and n.value == 566059

def vmsize():
    for line in open("/proc/self/status"):
        if line.startswith("VmSize:"):
            return int(line.split()[1]) * 1024

resource.setrlimit(resource.RLIMIT_AS, (vmsize() + (256 << 10), resource.RLIM_INFINITY))
rc = L.rd_build_states(12, None, ctypes.byref(n))
resource.setrlimit(resource.RLIMIT_AS, (resource.RLIM_INFINITY, resource.RLIM_INFINITY))
print("RC", rc, L.rd_last_error().decode())
rc2 = L.rd_build_states(12, None, ctypes.byref(n))
print("AFTER", rc2, n.value)
"""


def test_host_allocation_failure_is_enomem_not_abort(tmp_path):
    """rd.h: the C-ABI never aborts or throws.  With the address space capped just above what the
    process uses, the host word list of m = 12 (2.2 MB) cannot be allocated: the call returns
    RD_ENOMEM with a message instead of letting std::bad_alloc terminate the process, and the
    next call (limit lifted) succeeds."""
    import subprocess
    import sys
    f = tmp_path / "oom.py"
    f.write_text(OOM_SCRIPT)
    r = subprocess.run([sys.executable, str(f), ROOT], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr[-2000:]
    assert f"RC {rd.RD_ENOMEM} rd_build_states: host allocation failed" in r.stdout
    assert "AFTER 0 566059" in r.stdout


def test_every_status_entry_is_a_function_try_block():
    """Every C-ABI entry returning a status (int) in the library sources ends in RD_ABI_CATCH, so no
    C++ exception crosses the ABI (rd.h "Errors")."""
    import re
    csrc = os.path.join(ROOT, "paper_2409_17658_b200", "csrc")
    plain = {"rd_stats_len", "rd_stats_decide", "rd_chain_current_k", "rd_chain_gemm_variant"}   # accessors, no status
    for fn in ("rd_cuda.cu", "rd_host.cpp"):
        src = open(os.path.join(csrc, fn)).read()
        for mt in re.finditer(r'extern "C" int (rd_[a-z0-9_]+)\(', src):
            name = mt.group(1)
            if name in plain:
                continue
            body_start = src.index("{", mt.end())
            assert src[mt.end():body_start].rstrip().endswith("try"), name
            assert f'RD_ABI_CATCH("{name}")' in src, name


# Measured dense step times (ms, median of 10; m = 9 median of 3) of every (tile width, split)
# configuration on one B200 under the library's TMA policy (128-wide steps of >= 64 stages on
# TMA): "sN" every tile split N ways, "tailN" only the last partial wave's tiles
# (profiles/r02p_wave_probe_tma.txt).
WAVE_TABLE = {
    (6, 1): {"t128/s1": 0.0943, "t128/s2": 0.0674, "t128/s3": 0.0588, "t128/s4": 0.0726, "t64/s1": 0.0561,
             "t64/s2": 0.0634, "t64/s3": 0.0496, "t64/s4": 0.0536},
    (7, 1): {"t128/s1": 0.56, "t128/s2": 0.5687, "t128/s3": 0.5743, "t128/s4": 0.5477, "t128/tail2": 0.5733,
             "t128/tail3": 0.5723, "t128/tail4": 0.5497, "t128/tail5": 0.5478, "t128/tail6": 0.5595,
             "t64/s1": 0.5887, "t64/s2": 0.5569, "t64/s3": 0.5784, "t64/s4": 0.5744, "t64/tail2": 0.561,
             "t64/tail3": 0.5662, "t64/tail4": 0.5677, "t64/tail5": 0.5693, "t64/tail6": 0.5713},
    (7, 2): {"t128/s1": 0.381, "t128/s2": 0.3046, "t128/s3": 0.3378, "t128/s4": 0.3137, "t64/s1": 0.3049,
             "t64/s2": 0.3117, "t64/s3": 0.3154, "t64/s4": 0.2985},
    (7, 4): {"t128/s1": 0.2083, "t128/s2": 0.2184, "t128/s3": 0.2211, "t128/s4": 0.169, "t64/s1": 0.2098,
             "t64/s2": 0.1681, "t64/s3": 0.1847, "t64/s4": 0.1719},
    (8, 1): {"t128/s1": 11.0637, "t128/s2": 11.1431, "t128/s3": 11.2156, "t128/s4": 11.3022,
             "t128/tail2": 11.0173, "t128/tail3": 10.9731, "t128/tail4": 10.955, "t128/tail5": 10.9389,
             "t128/tail6": 10.9459, "t64/s1": 11.9874, "t64/s2": 11.9688, "t64/s3": 12.0615, "t64/s4": 12.0999,
             "t64/tail2": 11.8696, "t64/tail3": 11.9393, "t64/tail4": 11.9166, "t64/tail5": 11.8839,
             "t64/tail6": 11.8776},
    (8, 2): {"t128/s1": 5.7351, "t128/s2": 5.6232, "t128/s3": 5.661, "t128/s4": 5.6769, "t128/tail2": 5.5562,
             "t128/tail3": 5.551, "t128/tail4": 5.5501, "t128/tail5": 5.5437, "t128/tail6": 5.5469,
             "t64/s1": 6.0188, "t64/s2": 6.0595, "t64/s3": 6.0851, "t64/s4": 6.0697, "t64/tail2": 6.021,
             "t64/tail3": 6.0118, "t64/tail4": 5.9795, "t64/tail5": 5.9816, "t64/tail6": 5.9827},
    (8, 4): {"t128/s1": 2.9239, "t128/s2": 2.944, "t128/s3": 2.9649, "t128/s4": 2.9735, "t128/tail2": 2.9396,
             "t128/tail3": 2.9639, "t128/tail4": 2.9468, "t128/tail5": 2.9562, "t128/tail6": 2.9557,
             "t64/s1": 3.1636, "t64/s2": 3.1798, "t64/s3": 3.1922, "t64/s4": 3.2004, "t64/tail2": 3.1697,
             "t64/tail3": 3.1614, "t64/tail4": 3.1507, "t64/tail5": 3.1426, "t64/tail6": 3.1395},
    (8, 8): {"t128/s1": 1.9092, "t128/s2": 1.7086, "t128/s3": 1.6592, "t128/s4": 1.6296, "t128/tail2": 1.7042,
             "t128/tail3": 1.6433, "t128/tail4": 1.6208, "t128/tail5": 1.623, "t128/tail6": 1.6142,
             "t64/s1": 1.8614, "t64/s2": 1.7422, "t64/s3": 1.7098, "t64/s4": 1.7545, "t64/tail2": 1.7269,
             "t64/tail3": 1.6839, "t64/tail4": 1.7812, "t64/tail5": 1.7029, "t64/tail6": 1.687},
    (9, 8): {"t128/s1": 35.2239, "t128/s2": 35.3192, "t128/s3": 35.5107, "t128/s4": 35.7237,
             "t128/tail2": 35.0407, "t128/tail3": 34.837, "t128/tail4": 34.8145, "t128/tail5": 34.7571,
             "t128/tail6": 34.7664, "t64/s1": 39.3528, "t64/s2": 39.0722, "t64/s3": 39.0307, "t64/s4": 39.0456,
             "t64/tail2": 38.9533, "t64/tail3": 38.8235, "t64/tail4": 38.7639, "t64/tail5": 38.7282,
             "t64/tail6": 38.72},
}


def test_wave_model_picks_near_measured_best():
    """rd_dense_step_plan (the dense step's wave model, host only) picks, for every measured shape,
    a (tile width, split, split form) whose measured time is within 4 % of the best of the
    measured configurations (uniform splits 1..4, tail splits 2..6; profiles/r02p_wave_probe_tma.txt)
    (configuration-to-configuration noise is ~2 %), while the plain 128-tile step is up to 2x off."""
    from paper_2409_17658_b200 import dist as D
    worst_plain = 0.0
    for (m, p), t in WAVE_TABLE.items():
        N = rd.count_words(m)
        r0, r1 = D.panel_bounds(N, p, 0)
        tile, ns, tail, _ = rd.rd_dense_step_plan(r1 - r0, N)
        key = f"t{tile}/{'tail' if tail else 's'}{ns}"
        best = min(t.values())
        assert key in t, (m, p, key)
        assert t[key] <= 1.04 * best, (m, p, key, t[key], best)
        worst_plain = max(worst_plain, t["t128/s1"] / best)
    assert worst_plain > 1.9
    # forcing knobs reach the plan
    rd.rd_set_gemm_tile(128)
    rd.rd_set_split_k(0)
    try:
        assert rd.rd_dense_step_plan(848, 848)[:3] == (128, 1, False)
    finally:
        rd.rd_set_gemm_tile(0)
        rd.rd_set_split_k(1)
    with pytest.raises(rd.RDError):
        rd.rd_dense_step_plan(0, 848)
