"""Helpers for GPU tests: numpy <-> torch storage, oracle comparison."""
import numpy as np

import oracle

TORCH_DT = None


def torch_dtype(dtype):
    import torch
    return {"int32": torch.int32, "float32": torch.float32, "bfloat16": torch.bfloat16}[dtype]


def to_device(arr: np.ndarray, dtype: str, device):
    import torch
    if dtype == "bfloat16":
        return torch.from_numpy(arr.view(np.int16).copy()).to(device).view(torch.bfloat16)
    return torch.from_numpy(arr.copy()).to(device)


def to_numpy(t, dtype: str) -> np.ndarray:
    import torch
    t = t.detach().cpu()
    if dtype == "bfloat16":
        return t.view(torch.int16).numpy().view(np.uint16).copy()
    return t.numpy().copy()


def bits(a: np.ndarray) -> np.ndarray:
    return a.view(np.uint16 if a.itemsize == 2 else np.uint32)


def assert_parity(got: list, xs: list, N: int, G: int, dtype: str, what: str = ""):
    """Bit-exact vs the oracle (canonical order, R#7/R#8), all ranks equal,
    and within the north_star tolerance of the float64 / exact sum."""
    ref = oracle.lane_allreduce(xs, N, G, 1, dtype).out[0]
    for p, o in enumerate(got):
        if not np.array_equal(bits(o), bits(ref)):
            bad = np.nonzero(bits(o) != bits(ref))[0]
            raise AssertionError(f"{what} rank {p}: {len(bad)} mismatches, first at {bad[:8]}: "
                                 f"got {o[bad[:4]]} want {ref[bad[:4]]}")
    if dtype == "int32":
        assert np.array_equal(ref, oracle.brute_force_sum(xs, dtype))
    else:
        err = np.abs(oracle.to_float64(ref, dtype) - oracle.brute_force_sum(xs, dtype))
        assert np.all(err <= oracle.TOLERANCE[dtype] * oracle.abs_sum(xs, dtype) + 0.0)
