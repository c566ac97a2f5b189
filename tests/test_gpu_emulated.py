"""GPU parity of the CUDA path in emulated mode (``-m gpu``, one B200).

All P = N*G ranks run on one GPU through the C ABI
(lane_allreduce_init_emulated / lane_allreduce_emulated): the same kernel,
partition and cross-rank flag protocol as the multi-GPU path, launched as one
cooperative grid. Every output is compared element by element with the CPU
oracle on the same seeded inputs (bit-exact: int32 by definition, fp32/bf16
by the canonical order R#7/R#8), and the oracle with the float64 sum.
"""
import os

import numpy as np
import pytest

import oracle
import seeded_inputs as si
from tests.gpu_util import assert_parity, bits, to_device, to_numpy

pytestmark = pytest.mark.gpu

LAYOUTS = [(1, 2), (2, 1), (2, 2), (1, 4), (4, 1), (2, 4), (4, 2), (8, 1), (1, 8), (3, 1), (2, 3)]
COUNTS = [1, 7, 64, 4096 + 3, (1 << 18) + 5]
_COMMS = {}


@pytest.fixture(scope="module", autouse=True)
def _small_rounds():
    # 8 MiB of message per round keeps scratch small and makes the larger
    # counts run several rounds (kernel launches) per call
    old = {k: os.environ.get(k) for k in ("LANE_ROUND_BYTES", "LANE_TIMEOUT_MS")}
    os.environ["LANE_ROUND_BYTES"] = str(8 << 20)
    os.environ["LANE_TIMEOUT_MS"] = "5000"
    yield
    for c in _COMMS.values():
        c.close()
    _COMMS.clear()
    for k, v in old.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


def emu(N, G, k):
    import paper_2508_13397_b200 as lane
    key = (N, G, k, os.environ.get("LANE_ROUND_BYTES"), os.environ.get("LANE_CHUNK_BYTES"))
    if key not in _COMMS:
        _COMMS[key] = lane.LaneEmulator(N, G, k, device=0)
    return _COMMS[key]


def run(N, G, k, dtype, xs, inplace=False):
    import torch
    ins = [to_device(x, dtype, "cuda:0") for x in xs]
    outs = ins if inplace else [torch.full_like(t, 0) for t in ins]
    if not inplace:
        for o in outs:  # poison: every element must be written
            o.view(torch.int16 if dtype == "bfloat16" else torch.int32).fill_(-1)
    emu(N, G, k).allreduce(outs, ins)
    torch.cuda.synchronize()
    emu(N, G, k).check()
    return [to_numpy(o, dtype) for o in outs]


def test_seeded_fill_device_matches_numpy():
    import torch
    from seeded_inputs import device as sdev
    for dtype in ("int32", "float32", "bfloat16"):
        for dist in si.DISTS:
            t = torch.empty(10007, dtype={"int32": torch.int32, "float32": torch.float32,
                                          "bfloat16": torch.bfloat16}[dtype], device="cuda:0")
            sdev.fill(t, dtype, dist, 42, 3, start=123)
            torch.cuda.synchronize()
            ref = si.generate(dtype, dist, 42, 3, 10007, start=123)
            assert np.array_equal(bits(to_numpy(t, dtype)), bits(ref)), (dtype, dist)


@pytest.mark.parametrize("N,G", LAYOUTS)
@pytest.mark.parametrize("dtype", ["int32", "float32", "bfloat16"])
@pytest.mark.parametrize("mode", ["1", "2", "0"])
def test_parity_layouts(N, G, dtype, mode, monkeypatch):
    """LANE_DIRECT 1 = direct-pull (emulated default), 2 = direct-push (the
    registered multi-GPU job set), 0 = staged (the unregistered job set)."""
    monkeypatch.setenv("LANE_DIRECT", mode)
    for k in (1, 2, 4):
        for n in COUNTS:
            xs = si.generate_all(dtype, "signed", 42 + n, N * G, n)
            got = run(N, G, k, dtype, xs)
            assert_parity(got, xs, N, G, dtype, f"{N}x{G} k={k} n={n} mode={mode}")


@pytest.mark.parametrize("dtype", ["int32", "float32", "bfloat16"])
def test_parity_k_sweep_and_full_range(dtype):
    N, G = 2, 4
    dist = "full" if dtype == "int32" else "positive"
    for k in (1, 3, 8, 16):
        xs = si.generate_all(dtype, dist, 7, 8, 100003)
        assert_parity(run(N, G, k, dtype, xs), xs, N, G, dtype, f"k={k}")


@pytest.mark.parametrize("mode", ["1", "2", "0"])
def test_inplace_and_repeated_calls_epoch_reuse(mode, monkeypatch):
    monkeypatch.setenv("LANE_DIRECT", mode)
    N, G, k = 2, 4, 2
    for it in range(6):
        n = [5000, 1 << 16, 33, 1 << 20, 4097, 1 << 16][it]
        dtype = ["float32", "bfloat16", "int32"][it % 3]
        xs = si.generate_all(dtype, "signed", 100 + it, 8, n)
        got = run(N, G, k, dtype, xs, inplace=bool(it % 2))
        assert_parity(got, xs, N, G, dtype, f"iter {it}")


def test_multi_round_and_chunk_sizes():
    import paper_2508_13397_b200 as lane
    old = (os.environ.get("LANE_ROUND_BYTES"), os.environ.get("LANE_CHUNK_BYTES"))
    try:
        os.environ["LANE_ROUND_BYTES"] = str(1 << 20)  # 1 MiB per round
        os.environ["LANE_CHUNK_BYTES"] = str(16 << 10)
        c = emu(4, 2, 4)
        n = (3 << 20) // 4 + 11  # 3 MiB fp32 + a tail -> 4 rounds
        assert c.plan(n, "float32")["launches"] == 4
        xs = si.generate_all("float32", "signed", 9, 8, n)
        assert_parity(run(4, 2, 4, "float32", xs), xs, 4, 2, "float32", "multi-round")
    finally:
        for key, v in zip(("LANE_ROUND_BYTES", "LANE_CHUNK_BYTES"), old):
            if v is None:
                os.environ.pop(key, None)
            else:
                os.environ[key] = v


def test_p1_copy_and_zero_count():
    xs = si.generate_all("float32", "signed", 1, 1, 12345)
    assert np.array_equal(run(1, 1, 1, "float32", xs)[0], xs[0])
    import torch
    e = emu(2, 2, 1)
    z = [torch.empty(0, device="cuda:0") for _ in range(4)]
    e.allreduce(z, z)


def test_nan_positions_propagate():
    xs = si.generate_all("float32", "signed", 3, 8, 4099)
    xs[5][[0, 100, 4098]] = np.nan
    got = run(2, 4, 1, "float32", xs)
    for o in got:
        assert np.array_equal(np.isnan(o), np.isin(np.arange(4099), [0, 100, 4098]))


def test_errors_misaligned_and_dtype():
    import torch
    import paper_2508_13397_b200 as lane
    e = emu(2, 2, 1)
    base = [torch.zeros(1025, device="cuda:0") for _ in range(4)]
    mis = [b[1:] for b in base]  # 4-byte offset
    with pytest.raises(lane.LaneError) as ei:
        e.allreduce(mis, mis)
    assert ei.value.code == -6
    with pytest.raises(lane.LaneError) as ei:
        e.allreduce([b.double() for b in base], [b.double() for b in base])
    assert ei.value.code == -2


@pytest.mark.parametrize("piece", [None, 65536, 4096 * 3 + 16])
def test_host_buffer_api_emulated(piece):
    """lane_allreduce_emulated_host: pipelined H2D / kernel / D2H in pieces
    (each piece its own allreduce), including a ragged last piece."""
    import torch
    N, G = 2, 4
    old = os.environ.get("LANE_HOST_PIECE_BYTES")
    if piece:
        os.environ["LANE_HOST_PIECE_BYTES"] = str(piece)
    try:
        for dtype in ("float32", "bfloat16"):
            xs = si.generate_all(dtype, "signed", 11, 8, 300001)
            if dtype == "bfloat16":
                ins = [torch.from_numpy(x.view(np.int16).copy()).view(torch.bfloat16).pin_memory() for x in xs]
            else:
                ins = [torch.from_numpy(x).pin_memory() for x in xs]
            outs = [torch.empty_like(t).pin_memory() for t in ins]
            emu(N, G, 1).allreduce_host(outs, ins)
            assert_parity([to_numpy(o, dtype) for o in outs], xs, N, G, dtype, f"host api piece={piece}")
    finally:
        if old is None:
            os.environ.pop("LANE_HOST_PIECE_BYTES", None)
        else:
            os.environ["LANE_HOST_PIECE_BYTES"] = old


@pytest.mark.parametrize("N,G,k,dtype,n", [
    (2, 4, 1, "float32", 1 << 28),   # BASELINE configs[1] top size: 1 GiB per rank
    (4, 2, 4, "float32", 1 << 26),   # configs[2]: 256 MiB, k=4
    (8, 1, 1, "bfloat16", 1 << 28),  # configs[3]: bf16 512 MiB
])
def test_full_size_sampled_parity(N, G, k, dtype, n):
    """BASELINE sizes, default launch configuration (the one bench.py times):
    inputs filled on the device by the seeded generator; sampled outputs
    (every 4099th element, the last, and +-2 around every chunk/unit
    boundary) compared bit-exactly with the oracle run on those elements."""
    import torch
    import paper_2508_13397_b200 as lane
    from seeded_inputs import device as sdev
    old = os.environ.pop("LANE_ROUND_BYTES", None)
    try:
        c = lane.LaneEmulator(N, G, k, device=0)
        P = N * G
        tdt = {"float32": torch.float32, "bfloat16": torch.bfloat16}[dtype]
        ins = [sdev.fill(torch.empty(n, dtype=tdt, device="cuda:0"), dtype, "signed", 42, p) for p in range(P)]
        outs = [torch.empty_like(t) for t in ins]
        c.allreduce(outs, ins)
        torch.cuda.synchronize()
        c.check()
        plan = c.plan(n, dtype)
        units = oracle.partition(min(n, 1 << 22), 2 if dtype == "bfloat16" else 4, N, G, k,
                                 plan["chunk_granules"], plan["round_granules"])
        bnd = sorted({u.start for u in units} | {u.part_start for u in units})
        idx = si.sample_indices(n, 4099, bnd + [n - 1])
        xs = [si.generate_at(dtype, "signed", 42, p, idx) for p in range(P)]
        it = torch.from_numpy(idx).to("cuda:0")
        got = [to_numpy(o[it], dtype) for o in outs]
        assert_parity(got, xs, N, G, dtype, f"full {N}x{G} k={k} {dtype}")
        # all ranks identical over the WHOLE buffer (V1)
        for o in outs[1:]:
            assert torch.equal(o.view(torch.int16) if dtype == "bfloat16" else o.view(torch.int32),
                               outs[0].view(torch.int16) if dtype == "bfloat16" else outs[0].view(torch.int32))
        c.close()
        del ins, outs
        torch.cuda.empty_cache()
    finally:
        if old is not None:
            os.environ["LANE_ROUND_BYTES"] = old
