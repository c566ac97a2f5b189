"""Seeded, counter-based synthetic inputs for the lane allreduce.

This module is the ONE thing the oracle (``oracle/``) and the CUDA path share:
it holds no arithmetic of the method (no partition, no reduction, no rounding
of sums) — only the value generator. The CUDA side implements the same
counter-based generator independently in ``seeded_inputs/csrc/seeded_fill.cu``
(a bench/test utility, never called by the product path).

Generator (SURVEY.md §8(d) "Hash"):

    u(p, i) = mix64( mix64(seed ^ ((p + 1) * 0x9E3779B97F4A7C15)) ^ i )

``mix64`` is the SplitMix64 output function (state += golden gamma, then the
two xor-shift-multiply rounds). ``p`` is the rank, ``i`` the element index, so
any element of any rank's buffer can be regenerated on its own (sampled parity
at full size). Seed 42 is SPEC.md's default (S L468 [cli] "seed fixed default
42").

Distributions (paper is value-agnostic — "floats" with MPI_SUM, PAPER.md L312,
L341 — so values are chosen for exact reproducibility):

  int32  signed   ((u >> 43) mod 2^21) - 2^20          in [-2^20, 2^20)
  int32  full     int32(u >> 32)                        full range (wrap tests)
  fp32   signed   (((u >> 40) & 0xFFFFFF) - 2^23)*2^-23 in [-1, 1), exact
  fp32   positive 1 + ((u >> 41) & 0x7FFFFF)*2^-23      in [1, 2), exact
  bf16   signed   sign=u>>63, exp=119+((u>>56)&7), mant=(u>>49)&0x7F  (8 binades in [2^-8,1))
  bf16   positive exp=127, mant=(u>>49)&0x7F            in [1, 2)
  any    ones     1
  any    ramp     i mod 4096

bf16 values are returned as their uint16 bit patterns (numpy has no bf16).
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

DTYPES = ("int32", "float32", "bfloat16")
DISTS = ("signed", "positive", "full", "ones", "ramp")
# integer codes shared with the CUDA fill utility's C signature
DTYPE_CODE = {"int32": 0, "float32": 1, "bfloat16": 2}
DIST_CODE = {"signed": 0, "positive": 1, "full": 2, "ones": 3, "ramp": 4}
ITEMSIZE = {"int32": 4, "float32": 4, "bfloat16": 2}
NP_STORAGE = {"int32": np.int32, "float32": np.float32, "bfloat16": np.uint16}


def mix64(z):
    """SplitMix64 output function on uint64 (scalar or array), wrapping."""
    with np.errstate(over="ignore"):
        z = np.asarray(z, dtype=np.uint64) + GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def rank_key(seed: int, rank: int) -> np.uint64:
    with np.errstate(over="ignore"):
        k = np.uint64(seed) ^ (np.uint64(rank + 1) * GOLDEN)
    return mix64(k)


def hash_u64(seed: int, rank: int, idx) -> np.ndarray:
    idx = np.asarray(idx, dtype=np.uint64)
    return mix64(rank_key(seed, rank) ^ idx)


def values_from_hash(u: np.ndarray, idx: np.ndarray, dtype: str, dist: str) -> np.ndarray:
    """Map hash words to element values (storage dtype: int32 / float32 / uint16)."""
    u = np.asarray(u, dtype=np.uint64)
    idx = np.asarray(idx, dtype=np.uint64)
    if dist == "ones":
        if dtype == "int32":
            return np.ones(u.shape, np.int32)
        if dtype == "float32":
            return np.ones(u.shape, np.float32)
        return np.full(u.shape, 0x3F80, np.uint16)
    if dist == "ramp":
        r = (idx % np.uint64(4096)).astype(np.int64)
        if dtype == "int32":
            return r.astype(np.int32)
        if dtype == "float32":
            return r.astype(np.float32)
        # bf16 of an integer < 4096 needs rounding for > 256; use the exact
        # bf16-representable ramp (i mod 256) instead (documented in DESIGN.md)
        r = (idx % np.uint64(256)).astype(np.float32)
        return (r.view(np.uint32) >> np.uint32(16)).astype(np.uint16)
    if dtype == "int32":
        if dist == "full":
            return (u >> np.uint64(32)).astype(np.uint32).view(np.int32)
        v = ((u >> np.uint64(43)) % np.uint64(1 << 21)).astype(np.int64) - (1 << 20)
        return v.astype(np.int32)
    if dtype == "float32":
        if dist == "positive":
            m = ((u >> np.uint64(41)) & np.uint64(0x7FFFFF)).astype(np.float64)
            return (1.0 + m * 2.0 ** -23).astype(np.float32)
        m = ((u >> np.uint64(40)) & np.uint64(0xFFFFFF)).astype(np.float64)
        return ((m - 2.0 ** 23) * 2.0 ** -23).astype(np.float32)
    if dtype == "bfloat16":
        mant = ((u >> np.uint64(49)) & np.uint64(0x7F)).astype(np.uint16)
        if dist == "positive":
            return (np.uint16(127 << 7) | mant).astype(np.uint16)
        sign = (u >> np.uint64(63)).astype(np.uint16)
        exp = (np.uint64(119) + ((u >> np.uint64(56)) & np.uint64(7))).astype(np.uint16)
        return ((sign << np.uint16(15)) | (exp << np.uint16(7)) | mant).astype(np.uint16)
    raise ValueError(f"unknown dtype {dtype}")


def generate(dtype: str, dist: str, seed: int, rank: int, n: int, start: int = 0) -> np.ndarray:
    """Elements [start, start+n) of rank ``rank``'s buffer."""
    idx = np.arange(start, start + n, dtype=np.uint64)
    return values_from_hash(hash_u64(seed, rank, idx), idx, dtype, dist)


def generate_at(dtype: str, dist: str, seed: int, rank: int, indices) -> np.ndarray:
    """Elements at arbitrary indices of rank ``rank``'s buffer (sampled parity)."""
    idx = np.asarray(indices, dtype=np.uint64)
    return values_from_hash(hash_u64(seed, rank, idx), idx, dtype, dist)


def generate_all(dtype: str, dist: str, seed: int, P: int, n: int):
    return [generate(dtype, dist, seed, p, n) for p in range(P)]


def sample_indices(n: int, stride: int = 4099, boundaries=()) -> np.ndarray:
    """Sampled output positions: every ``stride``-th element, the last one, and
    +-2 around each given boundary (unit/chunk starts), clipped to [0, n)."""
    if n <= 0:
        return np.zeros(0, np.int64)
    s = set(range(0, n, stride))
    s.add(n - 1)
    for b in boundaries:
        for d in (-2, -1, 0, 1, 2):
            if 0 <= b + d < n:
                s.add(b + d)
    return np.array(sorted(s), dtype=np.int64)
