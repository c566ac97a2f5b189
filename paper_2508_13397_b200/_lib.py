"""ctypes loader for liblane_allreduce.so (the C ABI in include/lane_allreduce.h).

Argument marshalling only: every step of the allreduce runs in the library's
CUDA kernels. There is no fallback — if the shared library is missing this
module raises, on CPU and GPU hosts alike.
"""
from __future__ import annotations

import ctypes
import os
import re

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
# LANE_LIB_PATH: another build of THIS library (A/B measurements of kernel
# changes on one box); never a different implementation.
LIB_PATH = os.environ.get("LANE_LIB_PATH") or os.path.join(PKG, "liblane_allreduce.so")
HEADER = os.path.join(ROOT, "include", "lane_allreduce.h")

LANE_OK = 0
STATUS = {0: "LANE_OK", -1: "LANE_ERR_INVALID_ARG", -2: "LANE_ERR_UNSUPPORTED", -3: "LANE_ERR_CUDA",
          -4: "LANE_ERR_NOT_CONNECTED", -5: "LANE_ERR_TIMEOUT", -6: "LANE_ERR_MISALIGNED",
          -7: "LANE_ERR_MISMATCH"}
DTYPE = {"int32": 0, "float32": 1, "bfloat16": 2}
HANDLE_BYTES = 256
MAX_RANKS = 16


class LaneError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


_lib = None


def load() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2508_13397_b200.build` "
            "(the lane allreduce has no non-CUDA fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P, I, SZ, I64, U64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t, ctypes.c_int64, ctypes.c_uint64
    PP = ctypes.POINTER(ctypes.c_void_p)
    sig = {
        "lane_allreduce_init": (I, [I, I, I, PP]),
        "lane_allreduce_init_rank": (I, [I, I, I, I, I, PP]),
        "lane_allreduce_init_emulated": (I, [I, I, I, I, PP]),
        "lane_allreduce_get_handle": (I, [P, P, ctypes.POINTER(SZ)]),
        "lane_allreduce_open_peers": (I, [P, P, SZ]),
        "lane_allreduce": (I, [P, P, P, SZ, I, I, P]),
        "lane_allreduce_host": (I, [P, P, P, SZ, I, I, P]),
        "lane_allreduce_emulated": (I, [P, PP, PP, SZ, I, I, P]),
        "lane_allreduce_emulated_host": (I, [P, PP, PP, SZ, I, I, P]),
        "lane_allreduce_ring": (I, [P, P, P, SZ, I, I, P]),
        "lane_allreduce_ring_emulated": (I, [P, PP, PP, SZ, I, I, P]),
        "lane_allreduce_approach2": (I, [P, P, P, SZ, I, I, P]),
        "lane_allreduce_approach2_emulated": (I, [P, PP, PP, SZ, I, I, P]),
        "lane_allreduce_ring_plan": (I, [P, SZ, I, ctypes.POINTER(I64), ctypes.POINTER(I64),
                                         ctypes.POINTER(I), ctypes.POINTER(I)]),
        "lane_allreduce_finalize": (I, [P]),
        "lane_allreduce_register_handle": (I, [P, P, SZ, P, ctypes.POINTER(SZ)]),
        "lane_allreduce_register_open": (I, [P, P, SZ, ctypes.POINTER(I)]),
        "lane_allreduce_deregister": (I, [P, I]),
        "lane_allreduce_last_error": (ctypes.c_char_p, [P]),
        "lane_allreduce_check": (I, [P]),
        "lane_allreduce_trace": (I, [P, ctypes.POINTER(U64), SZ, ctypes.POINTER(SZ)]),
        "lane_allreduce_plan": (I, [P, SZ, I, ctypes.POINTER(I64), ctypes.POINTER(I64),
                                    ctypes.POINTER(I), ctypes.POINTER(I)]),
        "lane_allreduce_protocol": (I, [P, SZ, I, ctypes.POINTER(I)]),
        "lane_allreduce_ring_protocol": (I, [P, SZ, I, ctypes.POINTER(I)]),
        "lane_ll128_plan_query": (I, [I, I, I, I64, I, I64, I64, ctypes.POINTER(I64)]),
        "lane_ll128_line_query": (I, [I, I, I64, I64, I, I, I64, I, I64, ctypes.POINTER(I64)]),
        "lane_topology_query": (I, [I, I, I, ctypes.POINTER(I), ctypes.POINTER(I),
                                    ctypes.POINTER(I), ctypes.POINTER(I)]),
        "lane_partition_query": (I, [U64, I, I, I, I, I64, I64, ctypes.POINTER(I64), U64,
                                     ctypes.POINTER(U64)]),
        "lane_allreduce_version": (ctypes.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def header_symbols() -> list[str]:
    """Function names declared in include/lane_allreduce.h."""
    with open(HEADER) as f:
        text = f.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\**\s+\**(lane_\w+)\s*\(", text, flags=re.M)))


def check(code: int, comm=None) -> None:
    if code != LANE_OK:
        lib = load()
        msg = lib.lane_allreduce_last_error(comm)
        raise LaneError(code, (msg or b"").decode())
