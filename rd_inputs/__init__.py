"""Seeded synthetic inputs shared by the tests, bench.py and the oracle runs.

This module holds no arithmetic of the method (no (min,+) product, no words, no
matrix rules): only random operands with the shapes and value distributions of the
paper's workloads:

* ``operand``     uniform int16 in [lo, hi] with a fraction of +inf entries
                  (the generic rd_minplus_mul zoo: N up to C_9, inf density 0..1).
* ``power_like``  fully finite, entries in a band [c, c + 2m + 10] — the shape of
                  A^k for k >= 4.
* ``sparse_like`` density rho(m), labels 0..2m, inf elsewhere — the shape of A(G).
* ``sample_rows`` seeded row indices for sampled parity at full size.

Infinity is returned as the caller's sentinel (``inf``), so the same draw can feed
the oracle (int32, INT32_MAX) and the product (int16, 0x3FFF).
"""
from __future__ import annotations

import numpy as np

RHO = {1: 0.56, 2: 0.273, 3: 0.153, 4: 0.089, 5: 0.051, 6: 0.029, 7: 0.0168, 8: 0.0096, 9: 0.00553}


def operand(rows: int, cols: int, seed: int, inf_frac: float = 0.01, lo: int = 0, hi: int = 1000,
            inf: int = 0x3FFF, dtype=np.int16) -> np.ndarray:
    rng = np.random.default_rng(seed)
    X = rng.integers(lo, hi + 1, size=(rows, cols), dtype=np.int64)
    if inf_frac > 0:
        X[rng.random((rows, cols)) < inf_frac] = inf
    return X.astype(dtype)


def power_like(rows: int, cols: int, m: int, seed: int, base: int = 80, inf: int = 0x3FFF,
               dtype=np.int16) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.integers(base, base + 2 * m + 10 + 1, size=(rows, cols), dtype=np.int64).astype(dtype)


def sparse_like(n: int, m: int, seed: int, inf: int = 0x3FFF, dtype=np.int16) -> np.ndarray:
    rng = np.random.default_rng(seed)
    X = rng.integers(0, 2 * m + 1, size=(n, n), dtype=np.int64)
    X[rng.random((n, n)) >= RHO.get(m, 0.01)] = inf
    return X.astype(dtype)


def sample_rows(n: int, count: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    count = min(count, n)
    rows = rng.choice(n, size=count, replace=False)
    # always include the ragged tail and the first row
    return np.unique(np.concatenate([rows, [0, n - 1]])).astype(np.int64)


def to_inf(X: np.ndarray, src_inf: int, dst_inf: int, dtype) -> np.ndarray:
    """Re-encode the infinity sentinel (test marshalling between the two encodings)."""
    Y = X.astype(np.int64)
    Y[Y >= src_inf] = dst_inf
    return Y.astype(dtype)
