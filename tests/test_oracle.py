"""Pins for the CPU oracle (``-m "not gpu"``).

The oracle (oracle/lane_oracle.py) is checked against things other than
itself: the plain definition of allreduce (exact int64 sums, float64 sums),
its error bound, closed-form byte counts, special cases that reduce to a flat
sum, SPEC.md's printed worked examples (tests/golden/spec_examples.txt), a
hand-derived canonical-order fixture (tests/golden/canonical_order.txt), a
library rounding routine (torch's bf16 conversion) and a literal black-box
rendering of Alg. 2.
"""
import functools
import os

import numpy as np
import pytest

import oracle
import seeded_inputs as si
from oracle import lane_oracle as lo

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
LAYOUTS = [(1, 1), (1, 2), (2, 1), (1, 4), (2, 2), (4, 1), (1, 8), (2, 4), (4, 2), (8, 1),
           (1, 3), (3, 1), (2, 3)]


def _inputs(dtype, dist, P, n, seed=42):
    return si.generate_all(dtype, dist, seed, P, n)


# ---------------------------------------------------------------- SPEC examples
def _spec_lines():
    with open(os.path.join(GOLDEN, "spec_examples.txt")) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                yield line


def test_spec_split_examples():
    seen = 0
    for line in _spec_lines():
        if not line.startswith("split "):
            continue
        lhs, rhs = line.split("->")
        _, total, parts = lhs.split()
        lens, disp = rhs.split("|")
        lens = [int(v) for v in lens.split(",")]
        disp = [int(v) for v in disp.split(",")]
        got = oracle.split_remainder_first(int(total), int(parts))
        assert [ln for _, ln in got] == lens, line
        assert [s for s, _ in got] == disp, line
        seen += 1
    assert seen == 5


def test_spec_topology_examples():
    for line in _spec_lines():
        lhs, rhs = line.split("->")
        f = lhs.split()
        if f[0] == "world":
            N, G, k = map(int, f[1:4])
            t = oracle.Topology(N, G, k)
            assert t.P * t.procs_per_gpu == int(rhs), line
        elif f[0] == "rankinfo":
            N, G, k, r = map(int, f[1:5])
            t = oracle.Topology(N, G, k)
            p, l = divmod(r, k)  # spec rank = p*k + l (S L90 node-major, l_r minor)
            assert [t.node(p), t.gpu(p), l] == [int(v) for v in rhs.split()], line
        elif f[0] == "comms":
            N, G = map(int, f[1:3])
            t = oracle.Topology(N, G, 1)
            gs, ls = map(int, rhs.split())
            for p in range(t.P):
                assert len(t.comm_group(p)) == gs and len(t.comm_lane(p)) == ls
                # S L49: comm_group ∩ comm_lane = {p}
                assert set(t.comm_group(p)) & set(t.comm_lane(p)) == {p}


def test_spec_rs_ramp_example():
    # S L317: n=2 members, ramp count 4 -> member0 [0,2], member1 [4,6]
    xs = [np.arange(4, dtype=np.int32)] * 2
    res = oracle.lane_allreduce(xs, 1, 2, 1, "int32")
    assert res.T1[0].tolist() == [0, 2, 4, 6]


def test_spec_lane_ones_examples():
    n_cases = 0
    for line in _spec_lines():
        if not line.startswith("lane_ones"):
            continue
        lhs, rhs = line.split("->")
        N, G, k, n = map(int, lhs.split()[1:5])
        for dtype in ("int32", "float32", "bfloat16"):
            xs = _inputs(dtype, "ones", N * G, n)
            res = oracle.lane_allreduce(xs, N, G, k, dtype)
            for o in res.out:
                assert np.all(oracle.to_float64(o, dtype) == float(rhs)), line
        n_cases += 1
    assert n_cases == 3


def test_spec_stage2_chunk_example():
    # S L357: (2,4,2), count 2^10 -> stage-2 operand per rank per slice = 128
    for line in _spec_lines():
        if line.startswith("stage2_chunk"):
            lhs, rhs = line.split("->")
            N, G, k, n = map(int, lhs.split()[1:5])
            units = oracle.partition(n, 4, N, G, k)
            parts = {(u.l, u.g): u.part_end - u.part_start for u in units}
            assert len(parts) == k * G
            assert set(parts.values()) == {int(rhs)}


# ------------------------------------------------------- canonical-order fixture
def _parse_val(s, dtype):
    if dtype == "bfloat16":
        return np.uint16(int(s, 16))
    if dtype == "int32":
        return np.int32(int(s))
    return np.float32(float(s))


def _canonical_cases():
    with open(os.path.join(GOLDEN, "canonical_order.txt")) as f:
        for line in f:
            if line.startswith("case "):
                f_ = line.split()
                name, dtype, N, G, n = f_[1], f_[2], int(f_[3]), int(f_[4]), int(f_[5])
                ins = f_[6].split("=")[1].split(",")
                exp = f_[7].split("=")[1]
                yield name, dtype, N, G, n, [_parse_val(v, dtype) for v in ins], _parse_val(exp, dtype)


@pytest.mark.parametrize("case", list(_canonical_cases()), ids=lambda c: c[0])
@pytest.mark.parametrize("k", [1, 2])
def test_canonical_order_fixture(case, k):
    name, dtype, N, G, n, ins, exp = case
    xs = [np.full(n, v, dtype=lo.STORAGE[dtype]) for v in ins]
    res = oracle.lane_allreduce(xs, N, G, k, dtype)
    for o in res.out:
        assert np.all(o.view(np.uint32 if o.itemsize == 4 else np.uint16)
                      == np.array([exp]).view(np.uint32 if o.itemsize == 4 else np.uint16)), name


def test_canonical_fixture_count():
    assert len(list(_canonical_cases())) == 8


# ----------------------------------------------------------- plain definition
@pytest.mark.parametrize("N,G", LAYOUTS)
@pytest.mark.parametrize("n", [0, 1, 7, 64, 4099])
def test_int32_equals_exact_sum(N, G, n):
    """V2: int32 output == (sum_p int64 x_p) mod 2^32, any layout/k."""
    for dist in ("signed", "full"):
        xs = _inputs("int32", dist, N * G, n, seed=43)
        ref = oracle.brute_force_sum(xs, "int32")
        for k in (1, 2, 4):
            res = oracle.lane_allreduce(xs, N, G, k, "int32")
            for o in res.out:
                assert np.array_equal(o, ref)


def test_int32_matrix_spec_acceptance():
    """S L371/L516 oracle-equivalence matrix (nodes x gpus x ppg x counts)."""
    for N in (1, 2, 4, 8):
        for G in (1, 2, 4):
            for k in (1, 2, 4):
                for n in (1, 7, 64, 4096, 65536):
                    xs = _inputs("int32", "signed", N * G, n, seed=44)
                    ref = oracle.brute_force_sum(xs, "int32")
                    res = oracle.lane_allreduce(xs, N, G, k, "int32")
                    assert np.array_equal(res.out[-1], ref), (N, G, k, n)


@pytest.mark.parametrize("dtype", ["float32", "bfloat16"])
@pytest.mark.parametrize("dist", ["signed", "positive"])
@pytest.mark.parametrize("N,G", [(2, 4), (4, 2), (8, 1), (1, 8), (2, 2), (3, 1)])
def test_fp_within_error_bound(dtype, dist, N, G):
    """V3: |out - sum_f64| <= tol * sum|x|; fp32 also within the a-priori
    bound (P-1) * 2^-24 * sum|x| of P-1 correctly rounded adds."""
    P = N * G
    n = 1 << 14
    xs = _inputs(dtype, dist, P, n)
    ref = oracle.brute_force_sum(xs, dtype)
    mag = oracle.abs_sum(xs, dtype)
    res = oracle.lane_allreduce(xs, N, G, 1, dtype)
    err = np.abs(oracle.to_float64(res.out[0], dtype) - ref)
    assert np.all(err <= oracle.TOLERANCE[dtype] * mag)
    if dtype == "float32":
        assert np.all(err <= (P - 1) * 2.0 ** -24 * mag * (1 + 1e-12))
    else:
        # at most two roundings of 2^-8 relative each, plus fp32 adds
        bound = (2 * 2.0 ** -8 + (P - 1) * 2.0 ** -24) * mag * (1 + 1e-12)
        assert np.all(err <= bound)


def test_all_ranks_identical_and_deterministic():
    """V1 + determinism (S L228/L522)."""
    for dtype in ("int32", "float32", "bfloat16"):
        xs = _inputs(dtype, "signed", 8, 5000)
        r1 = oracle.lane_allreduce(xs, 2, 4, 2, dtype)
        r2 = oracle.lane_allreduce(xs, 2, 4, 2, dtype)
        for o in r1.out[1:]:
            assert o.tobytes() == r1.out[0].tobytes()
        assert r1.out[0].tobytes() == r2.out[0].tobytes()


# ------------------------------------------------------------- bf16 rounding pin
def test_bf16_rne_matches_torch():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(0)
    u = rng.integers(0, 2 ** 32, size=200000, dtype=np.uint64).astype(np.uint32)
    # add exact ties and near-ties, infinities, max values, zeros
    extra = np.array([0x3F808000, 0x3F818000, 0x3F807FFF, 0x3F808001, 0x7F7FFFFF, 0xFF7FFFFF,
                      0x7F800000, 0xFF800000, 0, 0x80000000, 0x00008000, 0x00018000], np.uint32)
    u = np.concatenate([u, extra])
    f = u.view(np.float32)
    finite = np.isfinite(f) | np.isinf(f)
    mine = oracle.bf16_round_nearest_even(f[finite])
    ref = torch.from_numpy(f[finite].copy()).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(mine, ref)
    nan = np.isnan(f)
    assert np.all(np.isnan((oracle.bf16_round_nearest_even(f[nan]).astype(np.uint32) << 16).view(np.float32)))


# ----------------------------------------------------------------- special cases
def _flat_sequential(xs, dtype):
    """A flat allreduce with one ascending-rank sum and one rounding: what the
    method reduces to with N = 1 (or G = 1)."""
    if dtype == "int32":
        return functools.reduce(np.add, [x.view(np.uint32) for x in xs]).view(np.int32)
    if dtype == "float32":
        return functools.reduce(np.add, [x.astype(np.float32) for x in xs])
    torch = pytest.importorskip("torch")
    acc = functools.reduce(np.add, [(x.astype(np.uint32) << 16).view(np.float32) for x in xs])
    return torch.from_numpy(acc).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)


@pytest.mark.parametrize("dtype", ["int32", "float32", "bfloat16"])
@pytest.mark.parametrize("P", [2, 3, 4, 8])
def test_single_node_and_single_gpu_reduce_to_flat_sum(dtype, P):
    """V6: N=1 is a flat RS+AG over G; G=1 is a flat allreduce over N (the
    'standard approach', P L335-349). Both equal one ascending flat sum."""
    xs = _inputs(dtype, "signed", P, 3001)
    ref = _flat_sequential(xs, dtype)
    for N, G in ((1, P), (P, 1)):
        for k in (1, 3):
            res = oracle.lane_allreduce(xs, N, G, k, dtype)
            for o in res.out:
                assert o.tobytes() == ref.tobytes(), (N, G, k)


@pytest.mark.parametrize("dtype", ["int32", "float32", "bfloat16"])
def test_p1_is_copy_and_empty(dtype):
    x = _inputs(dtype, "signed", 1, 777)
    res = oracle.lane_allreduce(x, 1, 1, 4, dtype)
    assert res.out[0].tobytes() == x[0].tobytes()
    res = oracle.lane_allreduce([np.zeros(0, lo.STORAGE[dtype])] * 8, 2, 4, 1, dtype)
    assert all(len(o) == 0 for o in res.out)


# ------------------------------------------------------------ invariance (V7)
@pytest.mark.parametrize("dtype", ["float32", "bfloat16"])
@pytest.mark.parametrize("N,G", [(2, 4), (4, 2), (8, 1)])
def test_k_and_chunk_invariance(dtype, N, G):
    xs = _inputs(dtype, "signed", N * G, 10007)
    base = oracle.lane_allreduce(xs, N, G, 1, dtype).out[0].tobytes()
    for k in (2, 4, 8):
        for cg in (None, 64, 1000):
            for rg in (None, 777):
                got = oracle.lane_allreduce(xs, N, G, k, dtype, cg, rg).out[0].tobytes()
                assert got == base, (k, cg, rg)


# ----------------------------------------------------- partition / ledger (V4, V5)
@pytest.mark.parametrize("n,itemsize,N,G,k,cg,rg", [
    (262144, 4, 2, 4, 1, None, None), (10, 4, 1, 4, 1, None, None), (1, 4, 2, 4, 8, None, None),
    (1000003, 4, 4, 2, 4, 4096, None), (1000003, 2, 8, 1, 8, 999, 70001), (7, 2, 2, 2, 2, 1, None),
    (64, 4, 1, 8, 8, None, None), (0, 4, 2, 2, 2, None, None), (4099, 4, 2, 4, 3, 5, 33)])
def test_partition_exactly_once(n, itemsize, N, G, k, cg, rg):
    units = oracle.partition(n, itemsize, N, G, k, cg, rg)
    cover = np.zeros(n, np.int64)
    q = 16 // itemsize
    for u in units:
        cover[u.start:u.end] += 1
        assert u.part_start <= u.start <= u.end <= u.part_end
        assert u.start % q == 0 or u.start == n  # units start on a 16-B granule (R#2)
    assert np.all(cover == 1)
    # every element is in exactly one group part per (round, l, c)
    parts = {(u.round, u.l, u.c, u.g): (u.part_start, u.part_end) for u in units}
    pc = np.zeros(n, np.int64)
    for s, e in parts.values():
        pc[s:e] += 1
    assert np.all(pc == 1)


@pytest.mark.parametrize("N,G", [(2, 4), (4, 2), (8, 1), (1, 8), (2, 2), (2, 1), (1, 2), (4, 1)])
@pytest.mark.parametrize("k", [1, 2, 4, 8])
def test_ledger_closed_forms(N, G, k):
    """V5: when n % (q*k*G*N) == 0 the ledger equals the closed forms
    phase1 (G-1)/G n, phase2 2(N-1)/N n/G, phase3 (G-1)/G n, total 2(P-1)/P n
    per rank per direction (north_star; SURVEY §8(a) totals)."""
    P = N * G
    q = 4
    n = q * k * G * N * 13
    xs = _inputs("int32", "ones", P, n)
    res = oracle.lane_allreduce(xs, N, G, k, "int32")
    L = res.ledger
    for p in range(P):
        for d in (L.recv, L.sent):
            assert d["phase1"][p] * G == (G - 1) * n
            assert (d["phase2_rs"][p] + d["phase2_ag"][p]) * N * G == 2 * (N - 1) * n
            assert d["phase3"][p] * G == (G - 1) * n
        assert L.total_recv()[p] * P == 2 * (P - 1) * n
        assert L.total_sent()[p] * P == 2 * (P - 1) * n
    # north_star: "2(G-1)/G n intra-node" and "per-lane n/G inter-node" volumes
    intra = L.recv["phase1"] + L.recv["phase3"]
    assert np.all(intra * G == 2 * (G - 1) * n)
    lane_operand = {(u.l, u.g): 0 for u in res.units}
    for u in res.units:
        lane_operand[(u.l, u.g)] += u.end - u.start
    per_g = [sum(v for (l, g), v in lane_operand.items() if g == gg) for gg in range(G)]
    assert all(v * G == n for v in per_g)


def test_ledger_uneven_equals_partition_sums():
    n, N, G, k = 4099, 2, 4, 3
    xs = _inputs("int32", "ones", 8, n)
    res = oracle.lane_allreduce(xs, N, G, k, "int32")
    exp = np.zeros(8, np.int64)
    for u in res.units:
        owner = u.a * G + u.g
        exp[owner] += (N - 1) * (u.end - u.start)
    assert np.array_equal(res.ledger.recv["phase2_rs"], exp)


def test_ownership_maps_complete():
    n = 5003
    res = oracle.lane_allreduce(_inputs("float32", "signed", 8, n), 2, 4, 2, "float32", 64)
    assert np.all(res.phase2_owner >= 0)
    assert np.all(res.phase1_owner >= 0)
    # phase-2 owner of an element is on its phase-1 owner's lane (same g)
    for a in range(2):
        assert np.all(res.phase1_owner[a] == res.phase2_owner % 4)


# ------------------------------------------------------ literal Alg. 2 (V8)
def _alg2_literal(xs64, N, G, k):
    """Alg. 2 per k-slice at offset s*l_r (P L346-348, L365) with black-box
    brute-force collectives: MPI_Reduce_scatter on comm_group, MPI_Allreduce
    on comm_lane, MPI_Allgatherv on comm_group (P L243-248). int64 arithmetic,
    element-granular remainder-first counts."""
    P = N * G
    n = len(xs64[0])
    buf_recv = [np.zeros(n, np.int64) for _ in range(P)]
    for l, (s0, sl) in enumerate(lo.split_remainder_first(n, k)):
        parts = lo.split_remainder_first(sl, G)  # c_ongroup, D
        for a in range(N):  # Reduce_scatter on comm_group of node a
            group = [a * G + h for h in range(G)]
            for r, p in enumerate(group):
                d, c = parts[r]
                buf_recv[p][s0 + d:s0 + d + c] = sum(xs64[q][s0 + d:s0 + d + c] for q in group)
        for g in range(G):  # Allreduce on comm_lane of GPU index g
            lane = [b * G + g for b in range(N)]
            d, c = parts[g]
            tot = sum(buf_recv[p][s0 + d:s0 + d + c] for p in lane)
            for p in lane:
                buf_recv[p][s0 + d:s0 + d + c] = tot
        for a in range(N):  # Allgatherv on comm_group
            group = [a * G + h for h in range(G)]
            for r, p in enumerate(group):
                d, c = parts[r]
                for q in group:
                    buf_recv[q][s0 + d:s0 + d + c] = buf_recv[p][s0 + d:s0 + d + c]
    return [((b & 0xFFFFFFFF).astype(np.uint32).view(np.int32)) for b in buf_recv]


@pytest.mark.parametrize("N,G,k", [(2, 4, 1), (2, 4, 2), (4, 2, 4), (8, 1, 1), (1, 4, 3), (3, 2, 2)])
def test_alg2_literal_cross_check(N, G, k):
    n = 1237
    xs = _inputs("int32", "full", N * G, n, seed=7)
    lit = _alg2_literal([x.astype(np.int64) for x in xs], N, G, k)
    ref = oracle.brute_force_sum(xs, "int32")
    res = oracle.lane_allreduce(xs, N, G, k, "int32")
    for p in range(N * G):
        assert np.array_equal(lit[p], ref)
        assert np.array_equal(res.out[p], lit[p])


# ------------------------------------------------------------------ errors
def test_topology_validation():
    for bad in ((0, 1, 1), (1, 0, 1), (1, 1, 0)):
        with pytest.raises(ValueError):
            oracle.Topology(*bad)
    with pytest.raises(ValueError):
        oracle.lane_allreduce([np.zeros(4, np.float32)] * 3, 2, 2, 1, "float32")
    with pytest.raises(ValueError):
        oracle.lane_allreduce([np.zeros(4, np.float32), np.zeros(5, np.float32)], 1, 2, 1, "float32")


def test_seeded_inputs_counter_based():
    a = si.generate("float32", "signed", 42, 3, 1000)
    b = si.generate_at("float32", "signed", 42, 3, [0, 17, 999])
    assert np.array_equal(a[[0, 17, 999]], b)
    assert np.all((a >= -1) & (a < 1))
    i = si.generate("int32", "signed", 42, 0, 100000)
    assert i.min() >= -(1 << 20) and i.max() < (1 << 20)
    h = si.generate("bfloat16", "signed", 42, 1, 100000)
    f = (h.astype(np.uint32) << 16).view(np.float32)
    assert np.all((np.abs(f) >= 2.0 ** -8) & (np.abs(f) < 1))
