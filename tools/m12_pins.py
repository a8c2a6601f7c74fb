"""m = 12 (outside SURVEY §8(f): NEXT-2 names m = 10, 11) — the round-1 opt-in pin kept as a
tool (~16 min on one B200): Cor 12 (26n/5 for 5 | n) and the row DP X3 for n = 3..10.
    python tools/m12_pins.py"""
import sys

sys.path.insert(0, ".")
import oracle as O  # noqa: E402
from paper_2409_17658_b200 import dist as rdist  # noqa: E402

def test_m12_panel_sequential_pins():
    # m = 12 (N = 566059) on one GPU, 26 panels: Cor 12 (26n/5 for 5 | n) and the
    # independent row DP X3 for n = 3..10; the conjectured (n0, 5, 26)
    from paper_2409_17658_b200 import dist as rdist
    got = rdist.power_sequence_panels(12, 45, alpha_max=5, panel_rows=22528, method=1)
    assert got["found"] and (got["alpha"], got["beta"]) == (5, 26)
    d = got["diag"]
    for n in range(5, got["k_stop"] + 1, 5):
        assert d[n] == 26 * n // 5, n
    for n in range(3, 11):
        assert d[n] == O.gamma_rowdp(12, n), n


if __name__ == "__main__":
    test_m12_panel_sequential_pins()
    print("m = 12 pins ok")
