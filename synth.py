"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

Holds none of the method's arithmetic: only the counter-based SplitMix64
generator of SURVEY.md C-5 (vectorised in numpy) and the input recipes built
from it.  The oracle (oracle/nb_oracle.c) and the CUDA path
(paper_2503_02134_b200/csrc) each carry their own implementation of the same
generator for the right-hand sides they build; this module exists so that test
inputs such as "a continuous random vector keyed by global id" come from one
place that neither side owns.
"""
from __future__ import annotations

import numpy as np

_M1 = np.uint64(0xD1B54A32D192ED03)
_G = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed: int, stream: int, ids) -> np.ndarray:
    ids = np.asarray(ids, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (np.uint64(seed) ^ (np.uint64(stream) * _M1)) + (ids + np.uint64(1)) * _G
        z ^= z >> np.uint64(30)
        z *= _C1
        z ^= z >> np.uint64(27)
        z *= _C2
        z ^= z >> np.uint64(31)
    return z


def uniform_by_id(seed: int, stream: int, ids) -> np.ndarray:
    """U(seed, stream, id) in [-1, 1), exact in double."""
    z = splitmix64(seed, stream, ids)
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53) * 2.0 - 1.0


def continuous_vector(gid: np.ndarray, mask: np.ndarray, seed: int = 0, stream: int = 4,
                      masked: bool = True) -> np.ndarray:
    """A continuous (equal on all copies of a node) random local vector."""
    v = uniform_by_id(seed, stream, gid)
    return v * mask if masked else v


def integer_field(n: int, seed: int = 0, stream: int = 6, lo: int = -64, hi: int = 64) -> np.ndarray:
    """Integer-valued local field (exact in every precision) for gather-scatter pins."""
    z = splitmix64(seed, stream, np.arange(n))
    return (lo + (z % np.uint64(hi - lo)).astype(np.int64)).astype(np.float64)
