"""The C-ABI from plain C: examples/rd_demo.c compiled with gcc against include/rd.h and
linked to librd.so (no Python in the loop)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2409_17658_b200")


def _build(tmp_path):
    exe = str(tmp_path / "rd_demo")
    subprocess.check_call(["gcc", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "examples", "rd_demo.c"), "-L", PKG, "-lrd",
                           f"-Wl,-rpath,{PKG}", "-o", exe])
    return exe


def test_c_demo_host_calls(tmp_path):
    out = subprocess.run([_build(tmp_path), "host"], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    assert "m=5: N=287 first=aaaaa last=ddddd nnz=4195" in out.stdout      # Table 1, V11
    assert "alpha=3 beta=2 d=(0,0,0)" in out.stdout                         # ceil(2n/3)
    assert "rd_build_matrix(0): -1" in out.stdout


@pytest.mark.gpu
def test_c_demo_gpu(tmp_path):
    out = subprocess.run([_build(tmp_path), "7", "100"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    assert "m=7: n0=21 alpha=5 beta=16" in out.stdout                       # Table 2
    assert "gamma_R(P_7 [] C_100) = 320" in out.stdout                      # 16n/5 for 5 | n
