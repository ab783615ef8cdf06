"""Synthetic point clouds for the benchmark configurations.

``uniform``   numpy PCG64 ``default_rng(seed).random((n, k), dtype=float32)``
              in [0, 1) -- the reference bench's distribution (cli.py:176-177)
              at float32.
``clustered`` 1024 centres ~U[0,1)^k (float32), cluster id ~U{0..1023},
              per-axis offset ~N(0, 0.01^2), point = centre + offset as
              float32.  Produces negative coordinates and dense regions.

Large inputs are generated in chunks seeded ``default_rng([seed, chunk])`` so
any prefix of the stream is reproducible without materialising the rest.
Variants used by the parity tests:
``ties``      floor(uniform * 64) / 64 (heavy duplication)
``signed_zero`` values drawn from {0.0, -0.0, 1.0, -1.0}
"""

from __future__ import annotations

import numpy as np

CHUNK = 1 << 24


def uniform(n: int, k: int, seed: int = 0) -> np.ndarray:
    if n <= CHUNK:
        return np.random.default_rng(seed).random((n, k), dtype=np.float32)
    out = np.empty((n, k), dtype=np.float32)
    for c, start in enumerate(range(0, n, CHUNK)):
        stop = min(n, start + CHUNK)
        out[start:stop] = np.random.default_rng([seed, c]).random((stop - start, k), dtype=np.float32)
    return out


def clustered(n: int, k: int, seed: int = 0, centres: int = 1024, sigma: float = 0.01) -> np.ndarray:
    rng = np.random.default_rng(seed)
    cen = rng.random((centres, k), dtype=np.float32)
    out = np.empty((n, k), dtype=np.float32)
    for c, start in enumerate(range(0, n, CHUNK)):
        stop = min(n, start + CHUNK)
        r = np.random.default_rng([seed, 1000 + c]) if n > CHUNK else rng
        ids = r.integers(0, centres, size=stop - start)
        off = r.normal(0.0, sigma, size=(stop - start, k)).astype(np.float32)
        out[start:stop] = cen[ids] + off
    return out


def ties(n: int, k: int, seed: int = 0, q: int = 64) -> np.ndarray:
    return (np.floor(uniform(n, k, seed) * q) / q).astype(np.float32)


def signed_zero(n: int, k: int, seed: int = 0) -> np.ndarray:
    vals = np.array([0.0, -0.0, 1.0, -1.0], dtype=np.float32)
    return vals[np.random.default_rng(seed).integers(0, 4, size=(n, k))]


GENERATORS = {
    "uniform": uniform,
    "clustered": clustered,
    "ties": ties,
    "signed_zero": signed_zero,
}


def make(kind: str, n: int, k: int, seed: int = 0) -> np.ndarray:
    return GENERATORS[kind](n, k, seed)
