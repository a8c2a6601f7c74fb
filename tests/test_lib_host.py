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
# configuration on one B200: "sN" every tile split N ways, "tailN" only the last partial wave's
# tiles (profiles/r02k_wave_probe.txt; "t128/s1" is cp.async, the TMA default is ~1 % faster).
WAVE_TABLE = {
    (6, 1): {"t128/s1": 0.0946, "t128/s2": 0.068, "t128/s3": 0.0602, "t128/s4": 0.0722, "t64/s1": 0.0546,
             "t64/s2": 0.0623, "t64/s3": 0.0484, "t64/s4": 0.0525},
    (7, 1): {"t128/s1": 0.5677, "t128/s2": 0.5887, "t128/s3": 0.5831, "t128/s4": 0.5549, "t128/tail2": 0.5871,
             "t128/tail3": 0.5896, "t128/tail4": 0.5707, "t128/tail5": 0.5569, "t128/tail6": 0.5683,
             "t64/s1": 0.5881, "t64/s2": 0.5569, "t64/s3": 0.576, "t64/s4": 0.5728, "t64/tail2": 0.5618,
             "t64/tail3": 0.5657, "t64/tail4": 0.5669, "t64/tail5": 0.5681, "t64/tail6": 0.5713},
    (7, 2): {"t128/s1": 0.3828, "t128/s2": 0.3077, "t128/s3": 0.3388, "t128/s4": 0.3153, "t64/s1": 0.305,
             "t64/s2": 0.3123, "t64/s3": 0.3112, "t64/s4": 0.2953},
    (7, 4): {"t128/s1": 0.2076, "t128/s2": 0.2206, "t128/s3": 0.2231, "t128/s4": 0.1684, "t64/s1": 0.2086,
             "t64/s2": 0.1673, "t64/s3": 0.1831, "t64/s4": 0.1708},
    (8, 1): {"t128/s1": 11.3724, "t128/s2": 11.4366, "t128/s3": 11.475, "t128/s4": 11.4517,
             "t128/tail2": 11.3652, "t128/tail3": 11.3566, "t128/tail4": 11.2752, "t128/tail5": 11.2868,
             "t128/tail6": 11.2931, "t64/s1": 12.0763, "t64/s2": 12.056, "t64/s3": 12.1472, "t64/s4": 12.1513,
             "t64/tail2": 11.9582, "t64/tail3": 12.0272, "t64/tail4": 12.0007, "t64/tail5": 11.9724,
             "t64/tail6": 11.9693},
    (8, 2): {"t128/s1": 5.9499, "t128/s2": 5.7553, "t128/s3": 5.8393, "t128/s4": 5.8014, "t128/tail2": 5.7285,
             "t128/tail3": 5.7746, "t128/tail4": 5.7175, "t128/tail5": 5.7057, "t128/tail6": 5.7102,
             "t64/s1": 6.0596, "t64/s2": 6.0967, "t64/s3": 6.124, "t64/s4": 6.0911, "t64/tail2": 6.0614,
             "t64/tail3": 6.0462, "t64/tail4": 6.0148, "t64/tail5": 6.0155, "t64/tail6": 6.0175},
    (8, 4): {"t128/s1": 3.0074, "t128/s2": 3.0181, "t128/s3": 3.0288, "t128/s4": 3.0382, "t128/tail2": 3.0321,
             "t128/tail3": 3.0361, "t128/tail4": 3.0258, "t128/tail5": 3.0213, "t128/tail6": 3.0207,
             "t64/s1": 3.1774, "t64/s2": 3.1951, "t64/s3": 3.207, "t64/s4": 3.1985, "t64/tail2": 3.1882,
             "t64/tail3": 3.1784, "t64/tail4": 3.1644, "t64/tail5": 3.1528, "t64/tail6": 3.1512},
    (8, 8): {"t128/s1": 2.0124, "t128/s2": 1.7782, "t128/s3": 1.7053, "t128/s4": 1.6705, "t128/tail2": 1.7708,
             "t128/tail3": 1.6911, "t128/tail4": 1.6583, "t128/tail5": 1.6501, "t128/tail6": 1.6654,
             "t64/s1": 1.8671, "t64/s2": 1.7468, "t64/s3": 1.713, "t64/s4": 1.7509, "t64/tail2": 1.732,
             "t64/tail3": 1.6879, "t64/tail4": 1.7227, "t64/tail5": 1.7054, "t64/tail6": 1.6889},
    (9, 8): {"t128/s1": 37.1532, "t128/s2": 37.1428, "t128/s3": 36.7907, "t128/s4": 36.9268,
             "t128/tail2": 37.0732, "t128/tail3": 36.674, "t128/tail4": 36.7436, "t128/tail5": 36.6013,
             "t128/tail6": 36.6432, "t64/s1": 39.6353, "t64/s2": 39.3649, "t64/s3": 39.3077, "t64/s4": 39.3118,
             "t64/tail2": 39.237, "t64/tail3": 39.109, "t64/tail4": 39.0526, "t64/tail5": 39.0353,
             "t64/tail6": 39.0334},
}


def test_wave_model_picks_near_measured_best():
    """rd_dense_step_plan (the dense step's wave model, host only) picks, for every measured shape,
    a (tile width, split, split form) whose measured time is within 4 % of the best of the
    measured configurations (uniform splits 1..4, tail splits 2..6; profiles/r02k_wave_probe.txt)
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
