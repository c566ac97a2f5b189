"""bench.py's in-run verification on CPU tensors (no GPU): ``sample_check``
accepts the method's exact outputs, rejects a one-element corruption, and with
LANE_PHASE2=ring (ring order per whole chunk, R#22) accepts the ring-variant
outputs by the exact-int / fp-tolerance rule."""
import os
import sys

import numpy as np
import pytest
import torch

import oracle
import seeded_inputs as si

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def _tensor(a, dtype):
    if dtype == "bfloat16":
        return torch.from_numpy(a.view(np.int16).copy()).view(torch.bfloat16)
    return torch.from_numpy(a.copy())


@pytest.mark.parametrize("dtype", ["int32", "float32", "bfloat16"])
def test_sample_check_direct(dtype, monkeypatch):
    monkeypatch.delenv("LANE_PHASE2", raising=False)
    N, G, n = 2, 4, 70001
    xs = si.generate_all(dtype, "signed", 42, N * G, n)
    out = _tensor(oracle.lane_allreduce(xs, N, G, 1, dtype).out[0], dtype)
    assert bench.sample_check([out], N, G, dtype, n, 42, [0])
    bad = out.clone()
    bad[n // 2] = bad[n // 2] + 1  # n // 2 is a sampled boundary
    assert not bench.sample_check([bad], N, G, dtype, n, 42, [0])


@pytest.mark.parametrize("dtype", ["int32", "float32", "bfloat16"])
def test_sample_check_ring_stage(dtype, monkeypatch):
    monkeypatch.setenv("LANE_PHASE2", "ring")
    N, G, n = 4, 1, 70001
    xs = si.generate_all(dtype, "signed", 42, N * G, n)
    out = _tensor(oracle.lane_allreduce(xs, N, G, 1, dtype, 4096, 1 << 20, phase2="ring").out[0], dtype)
    assert bench.sample_check([out], N, G, dtype, n, 42, [0])
    bad = out.clone()
    bad[n // 2] = bad[n // 2] + 1000
    assert not bench.sample_check([bad], N, G, dtype, n, 42, [0])


@pytest.mark.parametrize("N,G", [(1, 2), (2, 1), (2, 2), (2, 4), (4, 2), (8, 1), (1, 8), (3, 2)])
@pytest.mark.parametrize("dtype", ["int32", "float32", "bfloat16"])
def test_bench_canonical_sum_equals_oracle(N, G, dtype):
    """bench.py's own canonical-order reference (a few lines written from R#7 /
    R#8, no oracle import) and the oracle's step-by-step simulation agree bit
    for bit — two independent implementations of the same reading."""
    n = 5003
    xs = si.generate_all(dtype, "signed", 7, N * G, n)
    ref = oracle.lane_allreduce(xs, N, G, 2, dtype).out[0]
    got = bench.canonical_lane_sum(xs, N, G, dtype)
    vb = np.uint16 if dtype == "bfloat16" else np.uint32
    assert np.array_equal(np.asarray(got).view(vb), ref.view(vb))


@pytest.mark.parametrize("dtype", ["int32", "float32", "bfloat16"])
def test_ring_check(dtype):
    P, k, n = 4, 1, 9001
    xs = si.generate_all(dtype, "signed", 42, P, n)
    out = _tensor(oracle.ring_allreduce(xs, k, dtype, 4096, 1 << 20).out[0], dtype)
    assert bench.ring_check(out, P, k, dtype, n, 42, None)
    bad = out.clone()
    bad[7] = bad[7] + 1000
    assert not bench.ring_check(bad, P, k, dtype, n, 42, None)


@pytest.mark.parametrize("N,G", [(1, 2), (2, 1), (2, 2), (2, 4), (4, 2), (8, 1), (1, 8), (3, 2)])
@pytest.mark.parametrize("dtype", ["int32", "float32", "bfloat16"])
def test_bench_torch_canonical_sum_equals_oracle(N, G, dtype):
    """The torch form of the canonical order (the bench's whole-buffer device
    check) equals the oracle bit for bit, full-range int32 (wrap) included."""
    n = 5003
    dist = "full" if dtype == "int32" else "signed"
    xs = si.generate_all(dtype, dist, 11, N * G, n)
    ref = oracle.lane_allreduce(xs, N, G, 1, dtype).out[0]
    got = bench.canonical_lane_sum_torch([_tensor(x, dtype) for x in xs], N, G, dtype)
    vb = np.uint16 if dtype == "bfloat16" else np.uint32
    gb = got.view(torch.int16).numpy() if dtype == "bfloat16" else got.view(torch.int32).numpy()
    assert np.array_equal(gb.view(vb), ref.view(vb))


@pytest.mark.parametrize("dtype", ["int32", "float32", "bfloat16"])
def test_verify_whole_accepts_exact_rejects_any_flip(dtype):
    """verify_whole (chunked, every element) accepts the oracle's outputs for
    every rank and counts a single flipped element in the ragged last chunk."""
    N, G, n = 2, 2, 10007
    xs = si.generate_all(dtype, "signed", 42, N * G, n)
    ref = _tensor(oracle.lane_allreduce(xs, N, G, 1, dtype).out[0], dtype)

    def gen(p, s, m):
        return _tensor(si.generate(dtype, "signed", 42, p, m, start=s), dtype)

    outs = [ref.clone() for _ in range(N * G)]
    assert bench.verify_whole(outs, N, G, dtype, n, 42, chunk=4096, gen=gen) == (0, n * N * G)
    bad = outs[3]
    bad.view(torch.int16 if dtype == "bfloat16" else torch.int32)[n - 2] ^= 1
    assert bench.verify_whole(outs, N, G, dtype, n, 42, chunk=4096, gen=gen) == (1, n * N * G)
