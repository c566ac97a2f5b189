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
    key = (N, G, k) + tuple(os.environ.get(v) for v in ("LANE_ROUND_BYTES", "LANE_CHUNK_BYTES", "LANE_PROTO",
                                                        "LANE_LL_THRESHOLD_BYTES", "LANE_LL_CTAS",
                                                        "LANE_LL_MAX_BYTES", "LANE_PHASE2", "LANE_RING_CHUNK_BYTES",
                                                        "LANE_LL128_MIN_BYTES", "LANE_LL128_THRESHOLD_BYTES",
                                                        "LANE_LL128_MAX_BYTES", "LANE_DIRECT", "LANE_STORE",
                                                        "LANE_EMU_HANDSHAKE", "LANE_BULK_MIN_BYTES",
                                                        "LANE_DYN_CHUNKS", "LANE_CTAS_PER_GROUP",
                                                        "LANE_MIN_CHUNK_BYTES"))
    if key not in _COMMS:
        while len(_COMMS) >= 4:  # every emulated comm holds P ranks' scratch: keep a few
            _COMMS.pop(next(iter(_COMMS))).close()
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


def set_mode(mode, monkeypatch):
    """Simple-protocol job sets by LANE_DIRECT digit — 1 = direct-pull
    (emulated default), 2 = direct-push (the registered multi-GPU job set),
    3 = pull-all (registered, every job writes only its own rank's memory),
    4 = pull-push (registered: phase 1 reads the node's sendbufs, C and D push),
    0 = staged (the unregistered job set) — with suffix 'b' = TMA bulk stores
    (LANE_STORE=bulk: what every multi-GPU call >= LANE_BULK_MIN_BYTES runs)
    and 'h' = the start/end handshake with the call signature that every
    multi-GPU simple-protocol call runs (LANE_EMU_HANDSHAKE=1), 'd' = chunks
    claimed dynamically by the CTAs (LANE_DYN_CHUNKS=1); or the LL / LL128
    protocols."""
    if mode in ("ll", "ll128"):
        monkeypatch.setenv("LANE_PROTO", mode)
        return
    monkeypatch.setenv("LANE_PROTO", "simple")
    monkeypatch.setenv("LANE_DIRECT", mode[0])
    if "b" in mode:
        monkeypatch.setenv("LANE_STORE", "bulk")
    if "h" in mode:
        monkeypatch.setenv("LANE_EMU_HANDSHAKE", "1")
    if "d" in mode:
        monkeypatch.setenv("LANE_DYN_CHUNKS", "1")


@pytest.mark.parametrize("N,G", LAYOUTS)
@pytest.mark.parametrize("dtype", ["int32", "float32", "bfloat16"])
@pytest.mark.parametrize("mode", ["1", "2", "3", "4", "0", "ll", "ll128", "0hb", "2hb", "3hb", "4hb", "2h", "1b",
                                  "1d", "2hbd", "0hbd", "4hbd"])
def test_parity_layouts(N, G, dtype, mode, monkeypatch):
    """Every job set / store mode / protocol (set_mode) on every layout, k and
    ragged count, bit-exact vs the oracle."""
    set_mode(mode, monkeypatch)
    for k in (1, 2, 4):
        for n in COUNTS:
            if mode in ("ll", "ll128"):
                assert emu(N, G, k).protocol(n, dtype) == mode
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


@pytest.mark.parametrize("mode", ["1", "2", "3", "4", "0", "ll", "ll128", "mixed", "0hb", "2hb", "3hb", "4hb",
                                  "mixed-d", "1d"])
def test_inplace_and_repeated_calls_epoch_reuse(mode, monkeypatch):
    """Repeated calls of varying sizes reuse scratch, flags (fixed flag stride:
    one index, one meaning across calls), the handshake's control words and
    (LL, LL128) the two inbox parity sets; "mixed" alternates the LL, LL128 and
    simple protocols between calls ("mixed-d": with dynamic chunk claims, whose
    counters every kernel type zeroes one launch ahead)."""
    if mode.startswith("mixed"):
        if mode == "mixed-d":
            monkeypatch.setenv("LANE_DYN_CHUNKS", "1")
        monkeypatch.setenv("LANE_LL_THRESHOLD_BYTES", str(64 << 10))
        monkeypatch.setenv("LANE_LL128_MIN_BYTES", str(64 << 10))
        monkeypatch.setenv("LANE_LL128_THRESHOLD_BYTES", str(1 << 20))
    else:
        set_mode(mode, monkeypatch)
    N, G, k = 2, 4, 2
    for it in range(9):
        n = [5000, 1 << 16, 33, 1 << 20, 4097, 1 << 16, 9, 70001, 3][it]
        dtype = ["float32", "bfloat16", "int32"][it % 3]
        xs = si.generate_all(dtype, "signed", 100 + it, 8, n)
        got = run(N, G, k, dtype, xs, inplace=bool(it % 2))
        assert_parity(got, xs, N, G, dtype, f"iter {it}")
    if mode.startswith("mixed"):
        e = emu(N, G, k)
        assert e.protocol(5000, "float32") == "ll" and e.protocol(1 << 16, "float32") == "ll128"
        assert e.protocol(1 << 20, "float32") == "simple"


@pytest.mark.parametrize("ctas", ["1", "3", "37"])
def test_ll_cta_counts_and_chunking(ctas, monkeypatch):
    """LL protocol with few CTAs per rank (several chunks per CTA, phase-major
    within a CTA) and a message at the LL capacity's edge."""
    monkeypatch.setenv("LANE_PROTO", "ll")
    monkeypatch.setenv("LANE_LL_CTAS", str(int(ctas) * 8))
    for N, G, k in ((2, 4, 1), (4, 2, 2), (8, 1, 3), (1, 8, 1)):
        for n in (4097, (1 << 19) + 7):
            xs = si.generate_all("float32", "signed", 5 + n, 8, n)
            e = emu(N, G, k)
            assert e.protocol(n, "float32") == "ll"
            assert_parity(run(N, G, k, "float32", xs), xs, N, G, "float32", f"ll ctas={ctas} {N}x{G} k={k} n={n}")


@pytest.mark.parametrize("ctas", ["1", "5", "148"])
def test_ll128_cta_counts_and_sizes(ctas, monkeypatch):
    """LL128 protocol (lane_ll128.cuh): few CTAs per rank (several chunks per
    CTA, phase-major within a CTA; more lines per sub-part than a warp step
    covers), ragged sizes, and a message at the LL128 capacity's edge."""
    monkeypatch.setenv("LANE_PROTO", "ll128")
    monkeypatch.setenv("LANE_ROUND_BYTES", str(64 << 20))  # LL protocols run one-round messages only
    monkeypatch.setenv("LANE_LL_CTAS", str(int(ctas) * 8))
    monkeypatch.setenv("LANE_LL128_MAX_BYTES", str(16 << 20))
    for N, G, k in ((2, 4, 1), (4, 2, 2), (8, 1, 3), (1, 8, 1)):
        for n in (4097, (1 << 19) + 7, (4 << 20) - 3):
            xs = si.generate_all("float32", "signed", 5 + n, 8, n)
            e = emu(N, G, k)
            assert e.protocol(n, "float32") == "ll128"
            assert_parity(run(N, G, k, "float32", xs), xs, N, G, "float32", f"ll128 ctas={ctas} {N}x{G} k={k} n={n}")
    assert emu(2, 4, 1).protocol((4 << 20) + 4, "float32") == "simple"  # beyond the LL128 capacity


@pytest.mark.parametrize("N,G", [(1, 2), (2, 2), (2, 4), (8, 1)])
@pytest.mark.parametrize("dtype", ["float32", "bfloat16"])
def test_ll128_line_pair_positions(N, G, dtype, monkeypatch):
    """LL128 line pairs (15 granules per two lines, the pair's shared granule
    split across the two lane-7s): 40 consecutive ragged counts per layout,
    so the message's partial last granule, the sub-part ends and the chunk
    ends land on every position of a pair (0..14, including the shared
    granule 14) and sub-parts shorter than one pair occur; bit-exact vs the
    oracle on every rank."""
    monkeypatch.setenv("LANE_PROTO", "ll128")
    q = 4 if dtype == "float32" else 8
    P = N * G
    for k in (1, 2):
        e = emu(N, G, k)
        for m in range(40):
            n = q * (15 * P * 3 + 7 * m) + (m % q) + 1  # granules: 45P + 7m (+ a partial one)
            assert e.protocol(n, dtype) == "ll128"
            xs = si.generate_all(dtype, "signed", 300 + m, P, n)
            assert_parity(run(N, G, k, dtype, xs), xs, N, G, dtype, f"ll128 pairs {N}x{G} k={k} n={n}")


@pytest.mark.parametrize("N,G,dtype,mib", [(2, 4, "float32", 20), (4, 2, "bfloat16", 12), (1, 8, "float32", 10)])
def test_ll128_default_range_top_p8(N, G, dtype, mib, monkeypatch):
    """LL128 at the top of its default range on P = 8 layouts (2x4 takes LL128
    up to 32 MiB, 4x2 too, 1x8 up to 16 MiB), default chunking, a ragged
    tail: every element of every rank bit-exact vs the oracle."""
    monkeypatch.setenv("LANE_ROUND_BYTES", str(1 << 30))  # LL protocols run one-round messages only
    q = 4 if dtype == "float32" else 8
    n = (mib << 20) * q // 16 + 3
    e = emu(N, G, 1)
    assert e.protocol(n, dtype) == "ll128"
    xs = si.generate_all(dtype, "signed", 4242 + mib, N * G, n)
    assert_parity(run(N, G, 1, dtype, xs), xs, N, G, dtype, f"ll128 top {N}x{G} {mib} MiB")


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


@pytest.mark.parametrize("mode", ["1d", "2hbd", "0hbd"])
def test_dynamic_claims_multi_round_few_ctas(mode, monkeypatch):
    """Chunk claims (LANE_DYN_CHUNKS=1) with many chunks per CTA (3 or 6 CTAs
    per group; 8 ranks x k = 3 x 6 = 144 co-resident CTAs), k = 1 and 3, several rounds per call (each launch claims from
    its own zeroed counter), in-place and out-of-place: bit-exact vs the
    oracle on every rank."""
    set_mode(mode, monkeypatch)
    monkeypatch.setenv("LANE_ROUND_BYTES", str(4 << 20))
    monkeypatch.setenv("LANE_MIN_CHUNK_BYTES", str(16 << 10))
    monkeypatch.setenv("LANE_CHUNK_BYTES", str(64 << 10))
    for ctas in ("3", "6"):
        monkeypatch.setenv("LANE_CTAS_PER_GROUP", ctas)
        for N, G, k in ((2, 4, 1), (4, 2, 3), (1, 4, 1)):
            n = (9 << 20) // 4 + 13  # 9 MiB fp32 + a tail -> 3 rounds
            assert emu(N, G, k).plan(n, "float32")["launches"] == 3
            xs = si.generate_all("float32", "signed", 77 + k, N * G, n)
            got = run(N, G, k, "float32", xs, inplace=(ctas == "6"))
            assert_parity(got, xs, N, G, "float32", f"claims {mode} ctas={ctas} {N}x{G} k={k}")


@pytest.mark.filterwarnings("ignore:The CUDA Graph is empty")  # the refused host-API capture records nothing
def test_cuda_graph_capture_and_replay(monkeypatch):
    """Calls captured into a CUDA graph (simple, LL and LL128 protocols in one
    graph) replay correctly: every replay takes a fresh epoch from device
    memory. Inputs are refilled between replays, eager calls are interleaved
    with the replays, and every output is bit-exact vs the oracle; the
    host-buffer API refuses capture with LANE_ERR_UNSUPPORTED."""
    import torch
    import paper_2508_13397_b200 as lane
    from seeded_inputs import device as sdev
    monkeypatch.setenv("LANE_ROUND_BYTES", str(1 << 30))
    monkeypatch.setenv("LANE_LL128_THRESHOLD_BYTES", str(2 << 20))  # 4 MiB takes the simple protocol
    monkeypatch.setenv("LANE_LL_THRESHOLD_BYTES", str(64 << 10))
    N, G, k = 2, 4, 2
    P = N * G
    e = lane.LaneEmulator(N, G, k, device=0)  # fresh: graph mode is sticky per comm
    try:
        sizes = [(1 << 20) + 5, 3000, (1 << 18) + 3]  # simple (4 MiB), LL, LL128 (1 MiB)
        protos = [e.protocol(n, "float32") for n in sizes]
        assert protos == ["simple", "ll", "ll128"], protos
        ins = [[torch.empty(n, dtype=torch.float32, device="cuda:0") for _ in range(P)] for n in sizes]
        outs = [[torch.empty_like(t) for t in row] for row in ins]
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            g.capture_begin()
            for i_, o_ in zip(ins, outs):
                e.allreduce(o_, i_)
            g.capture_end()
        torch.cuda.current_stream().wait_stream(s)
        for rep in range(4):
            seed = 700 + rep
            for row in ins:
                for p, t in enumerate(row):
                    sdev.fill(t, "float32", "signed", seed, p)
            torch.cuda.synchronize()
            g.replay()
            torch.cuda.synchronize()
            e.check()
            for n, row in zip(sizes, outs):
                xs = si.generate_all("float32", "signed", seed, P, n)
                assert_parity([to_numpy(o, "float32") for o in row], xs, N, G, "float32", f"replay {rep} n={n}")
            # an eager call between replays (its epoch also comes from device memory now)
            n = 4099 + rep
            xs = si.generate_all("float32", "signed", 900 + rep, P, n)
            ein = [to_device(x, "float32", "cuda:0") for x in xs]
            eout = [torch.zeros_like(t) for t in ein]
            e.allreduce(eout, ein)
            torch.cuda.synchronize()
            assert_parity([to_numpy(o, "float32") for o in eout], xs, N, G, "float32", f"eager after replay {rep}")
        # the host-buffer API cannot be captured
        hin = [torch.zeros(1024, dtype=torch.float32).pin_memory() for _ in range(P)]
        hout = [torch.zeros_like(t).pin_memory() for t in hin]
        g2 = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            g2.capture_begin()
            try:
                with pytest.raises(lane.LaneError) as ei:
                    e.allreduce_host(hout, hin, stream=s)
            finally:
                g2.capture_end()
        assert ei.value.code == -2 and "capture" in str(ei.value)
    finally:
        e.close()


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
    boundary) compared bit-exactly with the oracle run on those elements,
    then every element of every rank against the device canonical-order sum."""
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
        # and the WHOLE buffer of every rank bit-exact against the canonical-order sum of the
        # regenerated inputs (bench.verify_whole on the device; pinned to the oracle bit for bit
        # by tests/test_bench_cpu.py)
        import bench
        bad, checked = bench.verify_whole(outs, N, G, dtype, n, 42)
        assert checked == n * P and bad == 0, (bad, checked)
        c.close()
        del ins, outs
        torch.cuda.empty_cache()
    finally:
        if old is not None:
            os.environ["LANE_ROUND_BYTES"] = old


def assert_ring_geometry(pl, chunk_bytes, round_bytes):
    """The ring's fp result depends on its pipeline chunk and round (R#21), so
    before the library's plan is handed to the oracle it must equal what R#21
    fixes from the environment the test set: chunk = LANE_RING_CHUNK_BYTES,
    round = LANE_LL_MAX_BYTES (in 16-byte granules). A planner that derived
    them from the launch configuration would otherwise be mirrored, not caught."""
    assert pl["chunk_granules"] == chunk_bytes // 16, pl
    assert pl["round_granules"] == round_bytes // 16, pl


def run_ring(N, G, k, dtype, xs, inplace=False):
    import torch
    ins = [to_device(x, dtype, "cuda:0") for x in xs]
    outs = ins if inplace else [torch.full_like(t, 0) for t in ins]
    if not inplace:
        for o in outs:
            o.view(torch.int16 if dtype == "bfloat16" else torch.int32).fill_(-1)
    emu(N, G, k).allreduce_ring(outs, ins)
    torch.cuda.synchronize()
    emu(N, G, k).check()
    return [to_numpy(o, dtype) for o in outs]


@pytest.mark.parametrize("P", [2, 3, 4, 8])
@pytest.mark.parametrize("dtype", ["int32", "float32", "bfloat16"])
@pytest.mark.parametrize("proto", ["ll", "ll128"])
def test_ring_parity(P, dtype, proto, monkeypatch):
    """Ring allreduce (Alg. 1, lane_allreduce_ring_emulated) vs the ring oracle,
    bit-exact: ring order per chunk, one rounding per hop — on the LL packets
    and on the LL128 lines (lane_ring_ll128_kernel)."""
    monkeypatch.setenv("LANE_PROTO", proto)
    for k in (1, 2, 3):
        for n in COUNTS:
            assert emu(1, P, k).ring_protocol(n, dtype) == proto
            xs = si.generate_all(dtype, "signed", 7 + n, P, n)
            got = run_ring(1, P, k, dtype, xs, inplace=(n % 2 == 1))
            pl = emu(1, P, k).plan(n, dtype, algorithm="ring")
            assert_ring_geometry(pl, 64 << 10, 16 << 20)  # R#21: fixed by the env, not the launch
            ref = oracle.ring_allreduce(xs, k, dtype, pl["chunk_granules"], pl["round_granules"]).out[0]
            for p, o in enumerate(got):
                assert np.array_equal(bits(o), bits(ref)), f"ring P={P} k={k} n={n} rank {p}"


@pytest.mark.parametrize("proto", ["ll", "ll128"])
def test_ring_multi_round_and_interleaved_with_lane(proto, monkeypatch):
    """Ring messages above the LL capacity run in several launches; ring and
    lane calls share the LL parity sets and the epoch counter."""
    monkeypatch.setenv("LANE_LL_MAX_BYTES", str(256 << 10))
    monkeypatch.setenv("LANE_PROTO", proto)
    N, G, k = 2, 2, 2
    for it, n in enumerate([(1 << 18) + 9, 1000, (1 << 16) + 1, 77]):
        dtype = ["float32", "int32", "bfloat16", "float32"][it]
        xs = si.generate_all(dtype, "signed", 50 + it, 4, n)
        got = run_ring(N, G, k, dtype, xs)
        pl = emu(N, G, k).plan(n, dtype, algorithm="ring")
        assert_ring_geometry(pl, 64 << 10, 256 << 10)
        assert pl["launches"] == -(-n * (2 if dtype == "bfloat16" else 4) // (256 << 10))
        ref = oracle.ring_allreduce(xs, k, dtype, pl["chunk_granules"], pl["round_granules"]).out[0]
        assert all(np.array_equal(bits(o), bits(ref)) for o in got), f"ring it={it}"
        got = run(N, G, k, dtype, xs)
        assert_parity(got, xs, N, G, dtype, f"lane it={it}")


@pytest.mark.parametrize("N,G", [(2, 2), (4, 2), (8, 1), (1, 8), (2, 4), (3, 2), (4, 1)])
@pytest.mark.parametrize("dtype", ["int32", "float32", "bfloat16"])
@pytest.mark.parametrize("proto", ["ll", "ll128"])
def test_lane_ring_phase2_parity(N, G, dtype, proto, monkeypatch):
    """LANE_PHASE2=ring: the lane method with Alg. 1 as the inter-node stage
    (fig:full_mpi_comparison) vs the oracle's ring variant, bit-exact, with
    small ring chunks and LL rounds so several chunks and launches occur —
    on the LL packets and on LL128 lines."""
    monkeypatch.setenv("LANE_PHASE2", "ring")
    monkeypatch.setenv("LANE_PROTO", proto)
    monkeypatch.setenv("LANE_RING_CHUNK_BYTES", str(8 << 10))
    monkeypatch.setenv("LANE_LL_MAX_BYTES", str(512 << 10))
    for k in (1, 3):
        for n in (1, 7, 4099, (1 << 17) + 5):
            assert emu(N, G, k).protocol(n, dtype) == proto
            xs = si.generate_all(dtype, "signed", 3 + n, N * G, n)
            got = run(N, G, k, dtype, xs, inplace=(n == 7))
            pl = emu(N, G, k).plan(n, dtype)
            assert_ring_geometry(pl, 8 << 10, 512 << 10)
            ref = oracle.lane_allreduce(xs, N, G, k, dtype, pl["chunk_granules"], pl["round_granules"],
                                        phase2="ring").out[0]
            for p, o in enumerate(got):
                assert np.array_equal(bits(o), bits(ref)), f"lane-ring {N}x{G} k={k} n={n} rank {p}"


@pytest.mark.parametrize("N,G", [(2, 2), (4, 2), (2, 4), (8, 1), (1, 8), (3, 2), (2, 3)])
@pytest.mark.parametrize("dtype", ["int32", "float32", "bfloat16"])
def test_approach2_parity(N, G, dtype, monkeypatch):
    """lane_allreduce_approach2_emulated ("approach 2", P L296-297) vs the
    approach-2 oracle — whose outputs are the lane method's bits — with small
    LL rounds so several launches and chunks occur."""
    import torch
    monkeypatch.setenv("LANE_LL_MAX_BYTES", str(512 << 10))
    for k in (1, 3):
        for n in (1, 7, 4099, (1 << 17) + 5):
            xs = si.generate_all(dtype, "signed", 11 + n, N * G, n)
            ins = [to_device(x, dtype, "cuda:0") for x in xs]
            outs = ins if n == 7 else [torch.full_like(t, 0) for t in ins]
            emu(N, G, k).allreduce_approach2(outs, ins)
            torch.cuda.synchronize()
            emu(N, G, k).check()
            ref = oracle.approach2_allreduce(xs, N, G, k, dtype).out[0]
            for p, o in enumerate(outs):
                assert np.array_equal(bits(to_numpy(o, dtype)), bits(ref)), f"a2 {N}x{G} k={k} n={n} rank {p}"


@pytest.mark.parametrize("N,G", [(2, 2), (4, 2), (1, 8), (8, 1)])
def test_lsu_engine_parity(N, G, monkeypatch):
    """LANE_ENGINE=lsu: the first (plain ld/st.global, phase-major) kernel, kept
    for A/B measurements — same partition, flags and canonical order."""
    monkeypatch.setenv("LANE_ENGINE", "lsu")
    monkeypatch.setenv("LANE_PROTO", "simple")
    import paper_2508_13397_b200 as lane
    e = lane.LaneEmulator(N, G, 2, device=0)
    try:
        import torch
        for dtype in ("int32", "float32", "bfloat16"):
            for n in (7, 4099, (1 << 18) + 5):
                xs = si.generate_all(dtype, "signed", 61 + n, N * G, n)
                ins = [to_device(x, dtype, "cuda:0") for x in xs]
                outs = [torch.full_like(t, 0) for t in ins]
                e.allreduce(outs, ins)
                torch.cuda.synchronize()
                e.check()
                assert_parity([to_numpy(o, dtype) for o in outs], xs, N, G, dtype, f"lsu {N}x{G} {dtype} n={n}")
    finally:
        e.close()


@pytest.mark.parametrize("proto", ["ll", "ll128"])
@pytest.mark.parametrize("k", [8, 16])
def test_ring_parity_ppg_8_16(proto, k, monkeypatch):
    """The paper's standard multi-PPG approach at its largest PPG (Alg. 1 on
    every k-slice, k up to 16, P L335-354, L431 "up to 16") on 8 emulated
    ranks (the 8-GPU box), both protocols, bit-exact vs the ring oracle."""
    monkeypatch.setenv("LANE_PROTO", proto)
    P = 8
    for dtype in ("float32", "bfloat16", "int32"):
        for n in (7, 4099, (1 << 18) + 5, (1 << 20) + 3):
            assert emu(1, P, k).ring_protocol(n, dtype) == proto
            xs = si.generate_all(dtype, "signed", 70 + n + k, P, n)
            got = run_ring(1, P, k, dtype, xs)
            pl = emu(1, P, k).plan(n, dtype, algorithm="ring")
            assert_ring_geometry(pl, 64 << 10, 16 << 20)
            ref = oracle.ring_allreduce(xs, k, dtype, pl["chunk_granules"], pl["round_granules"]).out[0]
            for p, o in enumerate(got):
                assert np.array_equal(bits(o), bits(ref)), f"ring P=8 k={k} {dtype} n={n} rank {p}"


@pytest.mark.parametrize("mode", ["1", "0hb", "2hb", "3hb", "4hb", "2h", "1d", "2hbd"])
@pytest.mark.parametrize("dtype", ["float32", "bfloat16"])
def test_whole_buffer_16mib_job_sets(mode, dtype, monkeypatch):
    """Every simple-protocol job set at 16 MiB per rank + a ragged tail (the
    size where the multi-GPU path switches to TMA bulk stores; default
    chunking, several chunks per CTA), 2x4, k = 2: EVERY element of every
    rank compared with the oracle (not sampled)."""
    monkeypatch.setenv("LANE_ROUND_BYTES", str(1 << 30))
    set_mode(mode, monkeypatch)
    N, G, k = 2, 4, 2
    n = (16 << 20) // (2 if dtype == "bfloat16" else 4) + 3
    xs = si.generate_all(dtype, "signed", 1600 + len(mode), N * G, n)
    e = emu(N, G, k)
    assert e.protocol(n, dtype) == "simple"
    assert_parity(run(N, G, k, dtype, xs), xs, N, G, dtype, f"16 MiB whole buffer mode={mode}")


def test_handshake_signature_agrees_across_calls(monkeypatch):
    """LANE_EMU_HANDSHAKE=1: the start handshake compares every rank's call
    signature; in a consistent call they agree (no LANE_ERR_MISMATCH) across
    sizes, dtypes and in-place calls, and the comm stays usable."""
    set_mode("2hb", monkeypatch)
    N, G, k = 4, 2, 1
    for it, n in enumerate([1 << 20, 33, (1 << 19) + 7, 1 << 20]):
        dtype = ["float32", "bfloat16", "int32", "float32"][it]
        xs = si.generate_all(dtype, "signed", 900 + it, N * G, n)
        assert_parity(run(N, G, k, dtype, xs, inplace=bool(it % 2)), xs, N, G, dtype, f"handshake it={it}")
    emu(N, G, k).check()


@pytest.mark.parametrize("mode", ["0hb", "2hb", "1h"])
def test_handshake_signature_mismatch_is_caught(mode, monkeypatch):
    """A call on which one rank disagrees (test hook LANE_EMU_SIG_SKEW_RANK:
    that rank publishes a different call signature, as a rank with unregistered
    buffers or other offsets would) stops in the start handshake on EVERY rank
    with LANE_ERR_MISMATCH — promptly (far below the 20 s watchdog), before any
    recvbuf is written — and the comm then refuses further calls."""
    import time
    import torch
    import paper_2508_13397_b200 as lane
    set_mode(mode, monkeypatch)
    monkeypatch.setenv("LANE_EMU_HANDSHAKE", "1")
    monkeypatch.setenv("LANE_EMU_SIG_SKEW_RANK", "3")
    monkeypatch.setenv("LANE_TIMEOUT_MS", "20000")
    N, G, n = 2, 4, (1 << 20) + 5
    e = lane.LaneEmulator(N, G, 2, device=0)  # not cached: the comm is poisoned afterwards
    try:
        xs = si.generate_all("float32", "signed", 5, N * G, n)
        ins = [to_device(x, "float32", "cuda:0") for x in xs]
        outs = [torch.full_like(t, 0).view(torch.int32).fill_(-1).view(torch.float32) for t in ins]
        t0 = time.time()
        e.allreduce(outs, ins)
        torch.cuda.synchronize()
        dt = time.time() - t0
        assert dt < 5.0, f"mismatch took {dt:.1f}s (watchdog instead of the signature check?)"
        with pytest.raises(lane.LaneError) as ei:
            e.check()
        assert ei.value.code == -7
        with pytest.raises(lane.LaneError) as ei:
            e.allreduce(outs, ins)
        assert ei.value.code == -7
        for o in outs:  # no recvbuf was touched
            assert bool((o.view(torch.int32) == -1).all())
    finally:
        e.close()


def test_host_api_staging_grows_between_calls(monkeypatch):
    """lane_allreduce_emulated_host with a small message and then larger ones
    on the SAME comm: the staging buffers grow while the copy streams and
    events stay valid (advisor finding: they used to be destroyed and reused)."""
    import torch
    import paper_2508_13397_b200 as lane
    monkeypatch.delenv("LANE_HOST_PIECE_BYTES", raising=False)
    N, G = 2, 2
    e = lane.LaneEmulator(N, G, 1, device=0)
    try:
        for it, n in enumerate([1000, 300001, (1 << 21) + 3, 5000]):
            xs = si.generate_all("float32", "signed", 300 + it, N * G, n)
            ins = [torch.from_numpy(x).pin_memory() for x in xs]
            outs = [torch.empty_like(t).pin_memory() for t in ins]
            e.allreduce_host(outs, ins)
            assert_parity([to_numpy(o, "float32") for o in outs], xs, N, G, "float32", f"host grow n={n}")
        with pytest.raises(lane.LaneError):
            e.allreduce_host([torch.empty(10) for _ in range(4)], [torch.empty(11) for _ in range(4)])
    finally:
        e.close()
