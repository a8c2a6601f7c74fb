"""Writes the oracle-derived golden files of tests/golden/ (test infrastructure).

Every value comes from oracle/ alone (no librd, no GPU); the tests compare the CUDA path with
these files.  Run:  python tools/make_golden.py [--m9] [--border]

  tests/golden/m9_power_hashes.json   64-bit BLAKE2b digests of every full power A^k, k = 1..27,
      of the m = 9 transfer matrix (N = C_9 = 21909), computed by the oracle's
      A^{k+1} = A^k (x) A with the INF terms skipped (the X4 form of the plain triple loop,
      SURVEY §8(c); Alg 2 step 3) — every power up to the detection power k* = 27 that
      Algorithm 2 step 4 compares entry by entry.  Digest input: the power as
      row-major little-endian int16, +inf written as RD_INF = 0x3FFF (rd.h's encoding).
  tests/golden/border_n11_rowdp.json  2 L_a(11) from the oracle's border row DP X7:
      the value at which P:664's "2 L_a(n) = n for 10 <= n <= 30" fails (R16).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")
RD_INF = 0x3FFF


def digest16(X: np.ndarray) -> str:
    """BLAKE2b-64 of X as row-major little-endian int16 with +inf -> 0x3FFF."""
    Y = np.where(X >= O.INF, RD_INF, X).astype("<i2")
    return hashlib.blake2b(np.ascontiguousarray(Y).tobytes(), digest_size=8).hexdigest()


def m9_hashes(kmax: int = 27):
    out = {}
    t0 = time.perf_counter()
    for k, X in O.powers(9, kmax):
        out[str(k)] = {"blake2b64": digest16(X), "n_inf": int((X >= O.INF).sum()),
                       "diag_min": int(O.diag_min(X))}
        print(f"m=9 k={k} {out[str(k)]} {time.perf_counter() - t0:.0f}s", flush=True)
    doc = {
        "_source": "oracle/ X4 chain (INF-skipping triple loop, SURVEY 8(c)) of A(G) for m = 9; "
                   "Alg 2 step 3 P:290, step 4 P:290-292; written by tools/make_golden.py",
        "encoding": "row-major little-endian int16, +inf = 0x3FFF, BLAKE2b digest_size 8",
        "m": 9, "N": O.count_words(9), "kmax": kmax, "powers": out,
    }
    with open(os.path.join(GOLDEN, "m9_power_hashes.json"), "w") as f:
        json.dump(doc, f, indent=1)


def border_n11():
    t0 = time.perf_counter()
    v = O.border_rowdp(11)
    doc = {
        "_source": "oracle/ border row DP X7 (2 L_a(n) = min_g 5g - 2|D(g)|, P:580-583) at n = 11; "
                   "P:664 claims 2 L_a(n) = n for 10 <= n <= 30 (DESIGN.md R16); written by tools/make_golden.py",
        "n": 11, "value": int(v), "seconds": round(time.perf_counter() - t0, 1),
    }
    with open(os.path.join(GOLDEN, "border_n11_rowdp.json"), "w") as f:
        json.dump(doc, f, indent=1)
    print(doc)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--m9", action="store_true")
    ap.add_argument("--border", action="store_true")
    a = ap.parse_args()
    O.build()
    if a.border or not a.m9:
        border_n11()
    if a.m9 or not a.border:
        m9_hashes()
