"""Counter-based Gaussian generator for the seeded synthetic signals.

Shared by the oracle side (tests, bench cpu_baseline) and the product side
(bench, smoke) as the ONLY common module: it holds no arithmetic of the
cascade method, just a reproducible map  (seed, stream, index) -> N(0,1).

Being counter-based, any window [start, start+count) of a signal can be
regenerated without materialising the rest, which is what the windowed
oracle needs for the 2^20-long E4 input.

Recipe (fixed):
  key   = splitmix64(seed * 0x9E3779B97F4A7C15 ^ (stream << 32))
  w1,w2 = splitmix64(key ^ (2*i)), splitmix64(key ^ (2*i + 1))
  u1    = ((w1 >> 11) + 0.5) * 2^-53         in (0, 1)
  u2    = (w2 >> 11) * 2^-53                 in [0, 1)
  z     = sqrt(-2 ln u1) * cos(2 pi u2)      (Box-Muller, cosine branch)
"""
from __future__ import annotations

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix64(x: np.ndarray) -> np.ndarray:
    x = (x + np.uint64(0x9E3779B97F4A7C15)) & _M64
    z = x
    z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & _M64
    z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & _M64
    return z ^ (z >> np.uint64(31))


def _key(seed: int, stream: int) -> np.uint64:
    with np.errstate(over="ignore"):
        s = (np.uint64(seed) * np.uint64(0x9E3779B97F4A7C15)) ^ (np.uint64(stream) << np.uint64(32))
        return _splitmix64(np.array([s], dtype=np.uint64))[0]


def normal(seed: int, stream: int, start: int, count: int) -> np.ndarray:
    """float64 N(0,1) samples for flat indices [start, start+count) of one stream."""
    if count <= 0:
        return np.zeros(0, dtype=np.float64)
    key = _key(seed, stream)
    i = np.arange(start, start + count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        w1 = _splitmix64(key ^ (i << np.uint64(1)))
        w2 = _splitmix64(key ^ ((i << np.uint64(1)) | np.uint64(1)))
    u1 = ((w1 >> np.uint64(11)).astype(np.float64) + 0.5) * (2.0 ** -53)
    u2 = (w2 >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)


def normal_chunked(seed: int, stream: int, start: int, count: int, out: np.ndarray,
                   chunk: int = 1 << 24) -> np.ndarray:
    """Fill a preallocated 1-D `out` (any float dtype) chunk by chunk (bounded host memory)."""
    done = 0
    while done < count:
        c = min(chunk, count - done)
        out[done:done + c] = normal(seed, stream, start + done, c)
        done += c
    return out
