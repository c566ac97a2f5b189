"""Pins for the ring allreduce oracle (oracle/ring_oracle.py, Alg. 1).

Checked against things other than itself: the plain definition (exact int64
sums mod 2^32; float64 sums within the per-hop error bound), the hand-derived
ring-order fixture tests/golden/ring_order.txt, closed-form byte and message
counts (2(p-1) messages, P L211; 2(P-1)/P*n elements per rank), and the P = 2
special case where one commutative add makes the ring and the lane method
bit-identical.
"""
import os

import numpy as np
import pytest

import oracle
import seeded_inputs as si
from oracle import lane_oracle as lo

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _cases(kind="case "):
    with open(os.path.join(GOLDEN, "ring_order.txt")) as f:
        for line in f:
            line = line.strip()
            if line.startswith(kind):
                yield line


def _val(s, dtype):
    return int(s, 16) if dtype == "bfloat16" else (float(s) if dtype == "float32" else int(s))


@pytest.mark.parametrize("line", list(_cases()))
def test_ring_order_fixture(line):
    f = line.split()
    name, dtype, P, n = f[1], f[2], int(f[3]), int(f[4])
    kv = dict(x.split("=") for x in f[5:])
    ins = [_val(v, dtype) for v in kv["inputs"].split(",")]
    exp = [_val(v, dtype) for v in kv["expect"].split(",")]
    own = [int(v) for v in kv["owners"].split(",")]
    xs = [np.full(n, v, dtype=lo.STORAGE[dtype]) for v in ins]
    r = oracle.ring_allreduce(xs, 1, dtype)
    q = 16 // lo.ITEMSIZE[dtype]
    for c, (e, o) in enumerate(zip(exp, own)):
        for p in range(P):
            got = r.out[p][c * q:(c + 1) * q]
            assert np.all(got == np.array(e, dtype=lo.STORAGE[dtype])), (name, c, p, got)
        assert np.all(r.owner[c * q:(c + 1) * q] == o), (name, c)


@pytest.mark.parametrize("P", [2, 3, 4, 8])
@pytest.mark.parametrize("k", [1, 3])
@pytest.mark.parametrize("n", [1, 5, 64, 4099])
def test_ring_int32_exact_and_identical(P, k, n):
    xs = si.generate_all("int32", "full", 3, P, n)
    r = oracle.ring_allreduce(xs, k, "int32")
    ref = oracle.brute_force_sum(xs, "int32")
    for o in r.out:
        assert np.array_equal(o, ref)


@pytest.mark.parametrize("dtype", ["float32", "bfloat16"])
@pytest.mark.parametrize("P", [3, 4, 8])
def test_ring_fp_error_bound(dtype, P):
    """fp32: P-1 RNE adds, |err| <= (P-1) 2^-24 sum|x|; bf16 adds one bf16
    rounding per hop (unit roundoff 2^-8 for 8 significant bits), |err| <=
    (P-1)(2^-24 + 2^-8) sum|x| (each hop's result
    is bounded by the partial sum of |x|)."""
    n = 20011
    xs = si.generate_all(dtype, "signed", 5, P, n)
    r = oracle.ring_allreduce(xs, 2, dtype)
    for o in r.out[1:]:
        assert np.array_equal(o.view(np.uint8), r.out[0].view(np.uint8))
    ref = oracle.brute_force_sum(xs, dtype)
    err = np.abs(oracle.to_float64(r.out[0], dtype) - ref)
    u = 2.0 ** -24 + (2.0 ** -8 if dtype == "bfloat16" else 0.0)
    assert np.all(err <= (P - 1) * u * oracle.abs_sum(xs, dtype) * (1 + 1e-9))


def test_ring_bf16_per_hop_differs_from_single_rounding():
    """R#11: the ring rounds every hop; the lane method rounds once per phase.
    On the fixture's inputs the two disagree (1.0 vs 1+2^-7)."""
    xs = [np.full(8, v, np.uint16) for v in (0x3F80, 0x3B80, 0x3B80)]
    ring = oracle.ring_allreduce(xs, 1, "bfloat16").out[0]
    lane = oracle.lane_allreduce(xs, 1, 3, 1, "bfloat16").out[0]
    assert ring[0] == 0x3F80 and lane[0] == 0x3F81


@pytest.mark.parametrize("P,k,n", [(2, 1, 4096), (4, 1, 4096), (8, 2, 1 << 14), (3, 1, 12)])
def test_ring_ledger_closed_forms(P, k, n):
    """Alg. 1 sends 2(p-1) messages (P L211); with n divisible by 4*k*P every
    rank sends and receives 2(P-1)/P * n elements."""
    xs = si.generate_all("int32", "signed", 1, P, n)
    r = oracle.ring_allreduce(xs, k, "int32")
    assert np.all(r.messages == 2 * (P - 1) * k)
    assert np.all(r.sent == 2 * (P - 1) * n // P)
    assert np.all(r.recv == 2 * (P - 1) * n // P)
    # chunk c completes on rank c-1 (the last rp of the reduce-scatter loop)
    for D in oracle.ring_chunks(n, 4, P, k):
        for c, (s, e) in enumerate(D):
            assert np.all(r.owner[s:e] == (c - 1) % P)


@pytest.mark.parametrize("dtype", ["float32", "bfloat16", "int32"])
def test_ring_p2_equals_lane(dtype):
    """P = 2: every element is one commutative add in both algorithms."""
    xs = si.generate_all(dtype, "signed", 9, 2, 777)
    ring = oracle.ring_allreduce(xs, 2, dtype).out[0]
    for N, G in ((1, 2), (2, 1)):
        lane = oracle.lane_allreduce(xs, N, G, 1, dtype).out[0]
        assert np.array_equal(ring.view(np.uint8), lane.view(np.uint8))


def test_ring_p1_and_empty():
    x = si.generate("float32", "signed", 1, 0, 33)
    assert np.array_equal(oracle.ring_allreduce([x], 1, "float32").out[0], x)
    r = oracle.ring_allreduce([np.zeros(0, np.float32)] * 3, 2, "float32")
    assert all(len(o) == 0 for o in r.out)


# ------------------------------------------------ lane method, ring inter-node stage
@pytest.mark.parametrize("line", list(_cases("lanering ")))
def test_lane_ring_phase2_fixture(line):
    f = line.split()
    dtype, N, G, n = f[2], int(f[3]), int(f[4]), int(f[5])
    kv = dict(x.split("=") for x in f[6:])
    ins = [_val(v, dtype) for v in kv["inputs"].split(",")]
    exp = [_val(v, dtype) for v in kv["expect"].split(",")]
    xs = [np.full(n, v, dtype=lo.STORAGE[dtype]) for v in ins]
    r = oracle.lane_allreduce(xs, N, G, 1, dtype, phase2="ring")
    q = 16 // lo.ITEMSIZE[dtype]
    for p in range(N * G):
        for gi, e in enumerate(exp):
            assert np.all(r.out[p][gi * q:(gi + 1) * q] == e), (p, gi)


@pytest.mark.parametrize("P", [3, 4, 8])
@pytest.mark.parametrize("dtype", ["float32", "bfloat16"])
def test_lane_ring_phase2_g1_is_alg1(P, dtype):
    """G = 1: no intra-node stage, one chunk per slice, the group part is the
    whole slice and its N sub-parts are exactly Alg. 1's chunks — the lane
    method with a ring inter-node stage IS the flat ring (two independently
    written simulations)."""
    xs = si.generate_all(dtype, "signed", 13, P, 5003)
    for k in (1, 2):
        a = oracle.lane_allreduce(xs, P, 1, k, dtype, phase2="ring").out[0]
        b = oracle.ring_allreduce(xs, k, dtype).out[0]
        assert np.array_equal(a.view(np.uint8), b.view(np.uint8))


@pytest.mark.parametrize("N,G", [(1, 4), (2, 4), (2, 2), (1, 8)])
def test_lane_ring_phase2_small_n_equals_direct(N, G):
    """N <= 2: at most one commutative add in the lane stage."""
    for dtype in ("float32", "bfloat16"):
        xs = si.generate_all(dtype, "signed", 21, N * G, 3001)
        a = oracle.lane_allreduce(xs, N, G, 2, dtype, phase2="ring")
        b = oracle.lane_allreduce(xs, N, G, 2, dtype)
        assert np.array_equal(a.out[0].view(np.uint8), b.out[0].view(np.uint8))


@pytest.mark.parametrize("N,G", [(4, 2), (8, 1), (3, 2), (4, 1)])
def test_lane_ring_phase2_exact_bound_and_ledger(N, G):
    P = N * G
    n = 16 * 3 * P * 8
    xs = si.generate_all("int32", "full", 2, P, n)
    r = oracle.lane_allreduce(xs, N, G, 3, "int32", phase2="ring")
    for o in r.out:
        assert np.array_equal(o, oracle.brute_force_sum(xs, "int32"))
    # same bytes as the direct stage: 2(P-1)/P * n per rank (V5)
    assert np.all(r.ledger.total_sent() == 2 * (P - 1) * n // P)
    for dtype in ("float32", "bfloat16"):
        xs = si.generate_all(dtype, "signed", 4, P, 4099)
        r = oracle.lane_allreduce(xs, N, G, 1, dtype, phase2="ring")
        err = np.abs(oracle.to_float64(r.out[0], dtype) - oracle.brute_force_sum(xs, dtype))
        u = 2.0 ** -24 + (2.0 ** -8 if dtype == "bfloat16" else 0.0)
        assert np.all(err <= P * u * oracle.abs_sum(xs, dtype) * (1 + 1e-9))


@pytest.mark.parametrize("dtype", ["float32", "bfloat16"])
def test_ring_pipeline_chunks_are_independent_rings(dtype):
    """R#21: with pipeline chunks every chunk is its own Alg. 1 ring — the
    chunked result equals running the unchunked ring on each chunk's elements
    (and the unchunked form on a single chunk), so only the chunk hierarchy,
    not the ring arithmetic, depends on the plan."""
    P, k, n, cg = 4, 2, 9001, 97
    q = 4 if dtype == "float32" else 8
    xs = si.generate_all(dtype, "signed", 17, P, n)
    full = oracle.ring_allreduce(xs, k, dtype, chunk_granules=cg).out[0]
    rings = oracle.ring_chunks(n, 16 // q, P, k, chunk_granules=cg)
    for D in rings:
        s, e = D[0][0], D[-1][1]
        if e > s:
            piece = oracle.ring_allreduce([x[s:e] for x in xs], 1, dtype).out[0]
            # the piece's own ring chunks match D only when the piece is granule-aligned (always, s % q == 0)
            assert np.array_equal(piece.view(np.uint8), full[s:e].view(np.uint8))
    # chunking changes the bits for fp (different ring start per element) but never int results
    xi = si.generate_all("int32", "full", 3, P, n)
    assert np.array_equal(oracle.ring_allreduce(xi, k, "int32", chunk_granules=cg).out[0],
                          oracle.brute_force_sum(xi, "int32"))


# ------------------------------------------------ "approach 2" (P L296-297)
@pytest.mark.parametrize("N,G", [(2, 4), (4, 2), (1, 8), (8, 1), (3, 2), (2, 2), (1, 1)])
@pytest.mark.parametrize("dtype", ["int32", "float32", "bfloat16"])
def test_approach2_outputs_equal_lane_method(N, G, dtype):
    """Node sum then lane sum, each in ascending order with one rounding: the
    same association as the lane method (R#7/R#8), so the outputs are
    bit-identical; int32 is also the exact sum."""
    xs = si.generate_all(dtype, "signed", 31, N * G, 4099)
    a = oracle.approach2_allreduce(xs, N, G, 2, dtype, chunk_granules=97)
    b = oracle.lane_allreduce(xs, N, G, 2, dtype).out[0]
    for o in a.out:
        assert np.array_equal(o.view(np.uint8), b.view(np.uint8))
    if dtype == "int32":
        assert np.array_equal(a.out[0], oracle.brute_force_sum(xs, dtype))


@pytest.mark.parametrize("N,G", [(2, 4), (4, 2), (1, 4), (4, 1)])
def test_approach2_ledger_closed_forms(N, G):
    """Per rank: (G-1)/G*n each way on node, (N-1)/N*n each way off node —
    every lane carries the whole buffer (vs n/G per lane for the lane method)."""
    P = N * G
    n = 4 * 3 * P * 64
    xs = si.generate_all("int32", "signed", 1, P, n)
    r = oracle.approach2_allreduce(xs, N, G, 3, "int32")
    assert np.all(r.sent["node_rs"] == (G - 1) * n // G) and np.all(r.sent["node_ag"] == (G - 1) * n // G)
    assert np.all(r.sent["lane_rs"] == (N - 1) * n // N) and np.all(r.sent["lane_ag"] == (N - 1) * n // N)
    lane = oracle.lane_allreduce(xs, N, G, 3, "int32").ledger.total_sent()
    assert np.all(sum(r.sent.values()) >= lane)
