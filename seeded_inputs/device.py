"""Device-side fill with the seeded generator (libseeded_fill.so).

The CUDA implementation is independent of the numpy one in ``__init__``; a
GPU test checks that both produce identical bits.
"""
from __future__ import annotations

import ctypes
import os

from . import DIST_CODE, DTYPE_CODE

LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libseeded_fill.so")
_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise ImportError(f"{LIB} missing: python -m paper_2508_13397_b200.build")
        _lib = ctypes.CDLL(LIB)
        _lib.seeded_fill.restype = ctypes.c_int
        _lib.seeded_fill.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int,
                                     ctypes.c_int, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p]
    return _lib


def fill(t, dtype: str, dist: str, seed: int, rank: int, start: int = 0, stream=None):
    """Fill CUDA tensor ``t`` (storage matching ``dtype``) with elements
    [start, start + t.numel()) of rank ``rank``'s seeded buffer."""
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    code = _load().seeded_fill(t.data_ptr(), t.numel(), start, DTYPE_CODE[dtype], DIST_CODE[dist], seed, rank,
                               int(s.cuda_stream))
    if code != 0:
        raise RuntimeError(f"seeded_fill failed: cudaError {code}")
    return t
