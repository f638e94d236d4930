"""Counter-based Gaussian generator for the seeded synthetic signals.

Shared by the oracle side (tests, bench cpu_baseline) and the product side (bench, smoke) as
the ONLY common module: it holds no arithmetic of the cascade method, just a reproducible map
(seed, stream, index) -> N(0,1) sample.

Being counter-based, any window [start, start+count) of a signal can be regenerated without
materialising the rest, which is what the windowed oracle needs
for the 2^20-long E4 input.

Recipe (fixed). For pair index j = i // 2:
  key   = splitmix64(seed * 0x9E3779B97F4A7C15 ^ (stream << 32))
  w     = splitmix64(key ^ j)
  u1    = ((w >> 40) + 0.5) * 2^-24          in (0, 1)       (float32)
  u2    = ((w >> 16) & 0xFFFFFF) * 2^-24      in [0, 1)       (float32)
  z_2j  = sqrt(-2 ln u1) cos(2 pi u2),  z_2j+1 = sqrt(-2 ln u1) sin(2 pi u2)   (float32)
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def _key(seed: int, stream: int) -> np.uint64:
    with np.errstate(over="ignore"):
        s = (np.uint64(seed) * np.uint64(0x9E3779B97F4A7C15)) ^ (np.uint64(stream) << np.uint64(32))
        return _splitmix64(np.array([s], dtype=np.uint64))[0]


def _pairs(key: np.uint64, j0: int, n: int) -> np.ndarray:
    """float32 samples for pair indices [j0, j0+n): returns 2n values (cos, sin interleaved)."""
    w = _splitmix64(key ^ np.arange(j0, j0 + n, dtype=np.uint64))
    u1 = ((w >> np.uint64(40)).astype(np.float32) + np.float32(0.5)) * np.float32(2.0 ** -24)
    u2 = ((w >> np.uint64(16)) & np.uint64(0xFFFFFF)).astype(np.float32) * np.float32(2.0 ** -24)
    r = np.sqrt(np.float32(-2.0) * np.log(u1))
    t = np.float32(2.0 * np.pi) * u2
    out = np.empty(2 * n, dtype=np.float32)
    out[0::2] = r * np.cos(t)
    out[1::2] = r * np.sin(t)
    return out


def normal32(seed: int, stream: int, start: int, count: int) -> np.ndarray:
    """float32 N(0,1) samples for flat indices [start, start+count) of one stream."""
    if count <= 0:
        return np.zeros(0, dtype=np.float32)
    key = _key(seed, stream)
    j0, j1 = start // 2, (start + count + 1) // 2
    vals = _pairs(key, j0, j1 - j0)
    off = start - 2 * j0
    return vals[off:off + count]


def normal(seed: int, stream: int, start: int, count: int) -> np.ndarray:
    """The same samples as float64 (exactly the float32 values, upcast)."""
    return normal32(seed, stream, start, count).astype(np.float64)


def normal_chunked(seed: int, stream: int, start: int, count: int, out: np.ndarray,
                   chunk: int = 1 << 22) -> np.ndarray:
    """Fill a preallocated 1-D float array with samples [start, start+count), in parallel chunks
    (numpy releases the GIL inside the vectorised kernels). Bit-identical to normal32()."""
    chunk -= chunk % 2
    offs = list(range(0, count, chunk))

    def work(o):
        c = min(chunk, count - o)
        out[o:o + c] = normal32(seed, stream, start + o, c)

    if len(offs) <= 1:
        for o in offs:
            work(o)
    else:
        with ThreadPoolExecutor(max_workers=min(len(offs), os.cpu_count() or 1)) as ex:
            list(ex.map(work, offs))
    return out
