"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic: it only draws matrix entries.
(SURVEY.md 8(c) c-xvi; BASELINE.json configs.)

* ``uniform(m, n, seed)``: entry (r, c) = u - 0.5 with u = top 53 bits of
  SplitMix64(seed, r + c*m) * 2**-53, i.e. U[-0.5, 0.5) exactly representable.
* ``normal(m, n, seed)``: Box-Muller on two such draws (host only; libm).

Matrices are returned column-major (Fortran order), dtype float64.
"""
from __future__ import annotations

import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

# Seeds proposed in SURVEY.md 8(d): 7073548 + config index (1-based).
SEED_BASE = 7073548


def _splitmix64(seed: int, idx: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + (idx + np.uint64(1)) * _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return z


def _u53(seed: int, start: int, count: int) -> np.ndarray:
    idx = np.arange(start, start + count, dtype=np.uint64)
    z = _splitmix64(seed, idx)
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def uniform(m: int, n: int, seed: int, chunk: int = 1 << 24) -> np.ndarray:
    """m x n column-major matrix, entries U[-0.5, 0.5)."""
    out = np.empty(m * n, dtype=np.float64)
    for s in range(0, m * n, chunk):
        c = min(chunk, m * n - s)
        out[s:s + c] = _u53(seed, s, c) - 0.5
    return out.reshape((m, n), order="F")


def normal(m: int, n: int, seed: int, chunk: int = 1 << 24) -> np.ndarray:
    """m x n column-major matrix, entries N(0,1) by Box-Muller on SplitMix64 draws.

    Element e uses draws 2e and 2e+1 of the stream: u1 in (0,1], u2 in [0,1).
    """
    out = np.empty(m * n, dtype=np.float64)
    for s in range(0, m * n, chunk):
        c = min(chunk, m * n - s)
        u = _u53(seed, 2 * s, 2 * c)
        u1 = 1.0 - u[0::2]
        u2 = u[1::2]
        out[s:s + c] = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)
    return out.reshape((m, n), order="F")


# BASELINE.json configs, in order (C1..C5).
CONFIGS = {
    "C1": dict(m=256, n=256, b=64, s=16, dist="uniform", seed=SEED_BASE + 1),
    "C2": dict(m=4096, n=4096, b=128, s=32, dist="uniform", seed=SEED_BASE + 2),
    "C3": dict(m=16384, n=16384, b=256, s=32, dist="uniform", seed=SEED_BASE + 3),
    "C4": dict(m=131072, n=2048, b=256, s=32, dist="normal", seed=SEED_BASE + 4),
    "C5": dict(m=65536, n=65536, b=512, s=64, dist="uniform", seed=SEED_BASE + 5),
}


def make(m: int, n: int, dist: str, seed: int) -> np.ndarray:
    if dist == "uniform":
        return uniform(m, n, seed)
    if dist == "normal":
        return normal(m, n, seed)
    raise ValueError(f"unknown distribution {dist!r}")


def checksum(a: np.ndarray) -> int:
    """64-bit wrapping sum of the matrix bytes viewed as uint64 (column-major)."""
    v = np.asfortranarray(a).reshape(-1, order="F").view(np.uint64)
    with np.errstate(over="ignore"):
        return int(np.add.reduce(v, dtype=np.uint64))
