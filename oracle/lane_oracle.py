"""CPU oracle for the k-split multi-lane allreduce of arXiv 2508.13397.

TEST INFRASTRUCTURE ONLY. Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module. The product path (``paper_2508_13397_b200/``) never imports it, and
this module imports nothing from the product path: the two share no code
(the seeded value generator in ``seeded_inputs/`` is the only shared module).

Citations: ``P Lnnn`` = PAPER.md line nnn; ``S Lnnn`` = SPEC.md line nnn;
``R#n`` = reading n in DESIGN.md §"Readings of the paper" (= SURVEY.md §8(c.3)).

What it computes
----------------
Plain definition (P L341 ``MPI_Allreduce(..., MPI_SUM, ...)``; S L538
glossary): every rank p ends with ``out_p[i] = sum_q x_q[i]``.

The method (Alg. 2 ``lane_allreduce``, P L218-251, applied per k-slice at
offset ``s*l_r`` as in §3.1/§3.1.2, P L328-373):

  O1 topology       rank p = a*G + g (node-major, R#6; S L90)
  O2 partition      16-byte granules; rounds -> k slices -> chunks -> G group
                    parts -> N lane sub-parts, remainder-first at every level
                    (R#2, R#3, R#4)
  O3 phase 1        intra-node reduce-scatter on comm_group (P L243):
                    T1_a[part g] = narrow(sum_{h=0..G-1} widen(x_{a,h}[part g]))
  O4 phase 2 RS     per-lane reduce on comm_lane (P L246, R#5):
                    F[U(g,a)] = narrow(sum_{b=0..N-1} widen(T1_b[U(g,a)]))
  O5 phase 2 AG     every lane member (b,g) receives F[U(g,a)] for all a
  O6 phase 3 AG     intra-node allgatherv on comm_group (P L248):
                    out_{a,g'}[part g] = R_{a,g}[part g]
  O7 outputs        per-rank outputs, per-rank per-phase ledger, ownership

Arithmetic (R#7, R#8, R#9): canonical ascending order (h then b), fp32
accumulation, int32 in wrap-around uint32, bf16 widened exactly to fp32 and
rounded to nearest-even ONCE per reducing phase.

Pinning: ``tests/test_oracle.py`` pins every function here against the plain
definition (brute-force int64 / float64 sums), error bounds, closed forms,
special cases, SPEC worked examples (``tests/golden/``) and a literal
black-box rendering of Alg. 2. The exact fp bit patterns are fixed by the
canonical-order reading R#7, which the paper leaves open; they are pinned by a
hand-computed fixture (``tests/golden/canonical_order.txt``).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

GRANULE_BYTES = 16  # R#2: partition unit, 16 B (one 128-bit vector)
ITEMSIZE = {"int32": 4, "float32": 4, "bfloat16": 2}
STORAGE = {"int32": np.int32, "float32": np.float32, "bfloat16": np.uint16}


# --------------------------------------------------------------------------
# O1 topology (P L330-332 new_comm; P L365 comm_group / comm_lane; S L44-51)
# --------------------------------------------------------------------------
@dataclass(frozen=True)
class Topology:
    nodes: int  # N
    gpus_per_node: int  # G
    procs_per_gpu: int  # k (CTA groups on B200; PPG in the paper)

    def __post_init__(self):
        for name in ("nodes", "gpus_per_node", "procs_per_gpu"):
            if int(getattr(self, name)) < 1:
                raise ValueError(f"{name} must be >= 1")  # S L57 "naming the field"

    @property
    def P(self) -> int:
        return self.nodes * self.gpus_per_node

    def node(self, p: int) -> int:
        return p // self.gpus_per_node

    def gpu(self, p: int) -> int:
        return p % self.gpus_per_node

    def rank(self, a: int, g: int) -> int:
        return a * self.gpus_per_node + g

    def comm_group(self, p: int) -> list[int]:
        """Ranks on p's node (same-node GPUs), ascending (S L49)."""
        a = self.node(p)
        return [self.rank(a, h) for h in range(self.gpus_per_node)]

    def comm_lane(self, p: int) -> list[int]:
        """Ranks with p's GPU index on every node, ascending (S L49)."""
        g = self.gpu(p)
        return [self.rank(b, g) for b in range(self.nodes)]


# --------------------------------------------------------------------------
# O2 partition (Alg. 2 c_group / c_ongroup / D, P L228-240; listing s/PPG at
# s*l_r, P L346-348; remainder-first rule S L160 lifted to granules, R#2)
# --------------------------------------------------------------------------
def split_remainder_first(total: int, parts: int) -> list[tuple[int, int]]:
    """(start, length) of ``parts`` contiguous pieces of ``total``: the first
    ``total % parts`` pieces get one extra (S L160, S L276-278)."""
    base, rem = divmod(total, parts)
    out = []
    start = 0
    for i in range(parts):
        ln = base + (1 if i < rem else 0)
        out.append((start, ln))
        start += ln
    return out


@dataclass(frozen=True)
class Unit:
    """One phase-2 ownership unit U(l, c, g, a) of one round (element range)."""

    round: int
    l: int  # k-slice ("process per GPU" l_r)
    c: int  # chunk within the slice
    g: int  # group part (phase-1 owner GPU index)
    a: int  # lane sub-part (phase-2 owner node index)
    part_start: int  # element range of group part (l, c, g)
    part_end: int
    start: int  # element range of the unit
    end: int


def partition(n: int, itemsize: int, N: int, G: int, k: int,
              chunk_granules: int | None = None,
              round_granules: int | None = None) -> list[Unit]:
    """All units, in (round, l, c, g, a) order.

    rounds: consecutive pieces of ``round_granules`` granules (last smaller);
    slices: remainder-first split of a round into k; chunks: consecutive pieces
    of ``chunk_granules`` granules of a slice (last smaller); group parts:
    remainder-first split of a chunk into G; sub-parts: remainder-first split
    of a group part into N. Granules are converted to elements and clipped at
    n (only the very last granule can be partial). ``None`` = one piece (the
    paper's one-shot partition)."""
    q = GRANULE_BYTES // itemsize
    ng = -(-n // q)
    units: list[Unit] = []
    if ng == 0:
        return units
    rg = ng if not round_granules else round_granules
    n_rounds = -(-ng // rg)

    def el(gr: int) -> int:
        return min(gr * q, n)

    for r in range(n_rounds):
        r0 = r * rg
        rlen = min(rg, ng - r0)
        for l, (s0, slen) in enumerate(split_remainder_first(rlen, k)):
            cg = slen if not chunk_granules else chunk_granules
            n_chunks = -(-slen // cg) if slen > 0 else 0
            for c in range(n_chunks):
                c0 = r0 + s0 + c * cg
                clen = min(cg, slen - c * cg)
                for g, (g0, glen) in enumerate(split_remainder_first(clen, G)):
                    ps, pe = c0 + g0, c0 + g0 + glen
                    for a, (u0, ulen) in enumerate(split_remainder_first(glen, N)):
                        us, ue = ps + u0, ps + u0 + ulen
                        units.append(Unit(r, l, c, g, a, el(ps), el(pe), el(us), el(ue)))
    return units


# --------------------------------------------------------------------------
# element arithmetic (R#7, R#8, R#9, R#12)
# --------------------------------------------------------------------------
def widen(v: np.ndarray, dtype: str) -> np.ndarray:
    """Exact widening to the accumulation type."""
    if dtype == "int32":
        return v.astype(np.int32).view(np.uint32)  # two's complement wrap (R#9)
    if dtype == "float32":
        return v.astype(np.float32)
    if dtype == "bfloat16":
        return (v.astype(np.uint32) << np.uint32(16)).view(np.float32)  # exact
    raise ValueError(dtype)


def bf16_round_nearest_even(f: np.ndarray) -> np.ndarray:
    """float32 -> bfloat16 bits, round to nearest, ties to even (R#8).
    NaN stays NaN (quiet bit set); payload is not part of parity (R#12)."""
    u = np.asarray(f, dtype=np.float32).view(np.uint32).astype(np.uint64)
    lsb = (u >> np.uint64(16)) & np.uint64(1)
    r = ((u + np.uint64(0x7FFF) + lsb) >> np.uint64(16)) & np.uint64(0xFFFF)
    nan = (u & np.uint64(0x7FFFFFFF)) > np.uint64(0x7F800000)
    r = np.where(nan, (u >> np.uint64(16)) | np.uint64(0x0040), r)
    return r.astype(np.uint16)


def narrow(acc: np.ndarray, dtype: str) -> np.ndarray:
    if dtype == "int32":
        return acc.astype(np.uint32).view(np.int32)
    if dtype == "float32":
        return acc.astype(np.float32)
    if dtype == "bfloat16":
        return bf16_round_nearest_even(acc)
    raise ValueError(dtype)


def add(acc: np.ndarray, v: np.ndarray, dtype: str) -> np.ndarray:
    """One accumulation step in the accumulation type (IEEE fp32 RNE / uint32
    wrap)."""
    with np.errstate(over="ignore"):
        return acc + v


# --------------------------------------------------------------------------
# ledger (O7; closed forms V5)
# --------------------------------------------------------------------------
@dataclass
class Ledger:
    """Per-rank element counts received/sent in each phase (bytes = x itemsize)."""

    P: int
    recv: dict = field(default_factory=dict)  # phase -> np.array[P]
    sent: dict = field(default_factory=dict)

    def __post_init__(self):
        for ph in ("phase1", "phase2_rs", "phase2_ag", "phase3"):
            self.recv[ph] = np.zeros(self.P, np.int64)
            self.sent[ph] = np.zeros(self.P, np.int64)

    def move(self, phase: str, src: int, dst: int, count: int):
        if src == dst:
            return
        self.sent[phase][src] += count
        self.recv[phase][dst] += count

    def total_recv(self) -> np.ndarray:
        return sum(self.recv.values())

    def total_sent(self) -> np.ndarray:
        return sum(self.sent.values())


@dataclass
class OracleResult:
    out: list  # per-rank output arrays (storage dtype)
    ledger: Ledger
    phase1_owner: np.ndarray  # [N, n] -> g that reduced element i on node a
    phase2_owner: np.ndarray  # [n] -> rank p = a*G+g that reduced element i
    units: list
    T1: list  # per-node phase-1 results (storage dtype), for intermediate pins
    F: np.ndarray  # phase-2 results (storage dtype)


# --------------------------------------------------------------------------
# the method, step by step
# --------------------------------------------------------------------------
def lane_allreduce(xs, N: int, G: int, k: int = 1, dtype: str = "float32",
                   chunk_granules: int | None = None,
                   round_granules: int | None = None,
                   phase2: str = "direct") -> OracleResult:
    """Simulate the P = N*G ranks of the k-split multi-lane allreduce.

    ``xs``: list of P input arrays (storage dtype: int32 / float32 / uint16 for
    bf16 bits), all of length n. Returns per-rank outputs plus the ledger and
    ownership maps. Follows O1-O7 above in the paper's phase order.

    ``phase2``: the lane stage's inner algorithm. "direct" (R#5): each owner
    reduces its sub-part over the lane in ascending b, then an allgather.
    "ring": the variant of fig:full_mpi_comparison (P L401, L457, "the ring
    algorithm is used in the inter-node stage"): Alg. 1 among the N lane
    members on every group part, whose N sub-parts are the ring chunks; ring
    chunk t starts on node t and completes on node t-1, one rounding per hop
    (R#11)."""
    topo = Topology(N, G, k)  # O1
    P = topo.P
    if len(xs) != P:
        raise ValueError(f"need {P} input buffers, got {len(xs)}")
    xs = [np.asarray(x, dtype=STORAGE[dtype]) for x in xs]
    n = len(xs[0])
    if any(len(x) != n for x in xs):
        raise ValueError("all ranks must pass the same count (P L341 collective semantics)")
    units = partition(n, ITEMSIZE[dtype], N, G, k, chunk_granules, round_granules)  # O2
    ledger = Ledger(P)
    phase1_owner = np.full((N, n), -1, np.int64)
    phase2_owner = np.full(n, -1, np.int64)

    # group parts (l, c, g) of every round; each is the union of its N units
    parts = {}
    for u in units:
        parts.setdefault((u.round, u.l, u.c, u.g), (u.part_start, u.part_end))

    # O3 phase 1: intra-node reduce-scatter (P L243; P L365-368). On every
    # node a, GPU g reduces group part g over the G ranks of comm_group in
    # ascending h (R#7), one rounding (R#8).
    T1 = [np.zeros(n, STORAGE[dtype]) for _ in range(N)]
    for (_, _, _, g), (s, e) in parts.items():
        for a in range(N):
            owner = topo.rank(a, g)
            acc = widen(xs[topo.rank(a, 0)][s:e], dtype)
            for h in range(1, G):
                acc = add(acc, widen(xs[topo.rank(a, h)][s:e], dtype), dtype)
            T1[a][s:e] = narrow(acc, dtype)
            phase1_owner[a, s:e] = g
            for h in range(G):
                ledger.move("phase1", topo.rank(a, h), owner, e - s)

    # O4 phase 2 reduce-scatter on comm_lane (P L246, R#5): the owner (a, g)
    # of unit U(g, a) sums T1 of every node b in ascending b, one rounding.
    F = np.zeros(n, STORAGE[dtype])
    if phase2 == "ring":
        _phase2_ring(T1, F, units, topo, dtype, ledger, phase2_owner)
    elif phase2 != "direct":
        raise ValueError(phase2)
    for u in units if phase2 == "direct" else []:
        s, e = u.start, u.end
        owner = topo.rank(u.a, u.g)
        acc = widen(T1[0][s:e], dtype)
        for b in range(1, N):
            acc = add(acc, widen(T1[b][s:e], dtype), dtype)
        F[s:e] = narrow(acc, dtype)
        phase2_owner[s:e] = owner
        for b in range(N):
            ledger.move("phase2_rs", topo.rank(b, u.g), owner, e - s)

    # O5 phase 2 allgather on comm_lane: every (b, g) receives F[U(g, a)].
    # (ring variant: the ring's allgather loop, ledger in _phase2_ring)
    # R[p] is rank p's copy of its group parts after the lane allreduce
    # (Alg. 2: "MPI_Allreduce to buf_recv at offset r(c_group)", P L246).
    SENT = _sentinel(dtype)
    R = [np.full(n, SENT, STORAGE[dtype]) for _ in range(P)]
    for u in units:
        s, e = u.start, u.end
        owner = phase2_owner[s] if e > s else topo.rank(u.a, u.g)
        for b in range(N):
            dst = topo.rank(b, u.g)
            R[dst][s:e] = F[s:e]
            if phase2 == "direct":
                ledger.move("phase2_ag", owner, dst, e - s)

    # O6 phase 3: intra-node allgatherv on comm_group (P L248, "using D"):
    # rank (a, g') receives group part g from (a, g) for every g.
    out = [np.full(n, SENT, STORAGE[dtype]) for _ in range(P)]
    for (_, _, _, g), (s, e) in parts.items():
        for a in range(N):
            src = topo.rank(a, g)
            for gp in range(G):
                dst = topo.rank(a, gp)
                out[dst][s:e] = R[src][s:e]
                ledger.move("phase3", src, dst, e - s)

    return OracleResult(out, ledger, phase1_owner, phase2_owner, units, T1, F)


def _phase2_ring(T1, F, units, topo, dtype, ledger, phase2_owner):
    """O4+O5, ring variant: Alg. 1 (P L150-206) on comm_lane for every group
    part. The part's N units (sub-parts a = 0..N-1) are the ring chunks.
    Reduce-scatter step i: node b sends chunk b-i to b+1, which adds its own
    T1 chunk in ONE rounding (MPI_Reduce); chunk t therefore accumulates
    T1_t, T1_{t+1}, ..., T1_{t-1} and completes on node t-1. The allgather
    loop then gives every lane member every chunk (N-1 steps)."""
    N = topo.nodes
    groups = {}
    for u in units:
        groups.setdefault((u.round, u.l, u.c, u.g), []).append(u)
    for (_, _, _, g), us in groups.items():
        for t, u in enumerate(us):  # ring chunk t = sub-part a = t
            s, e = u.start, u.end
            cur = T1[t][s:e].copy()
            for i in range(1, N):
                b = (t + i) % N  # the node that receives the partial from b-1 and adds its own
                cur = narrow(add(widen(cur, dtype), widen(T1[b][s:e], dtype), dtype), dtype)
            F[s:e] = cur
            phase2_owner[s:e] = topo.rank((t - 1) % N, g)
        # ledger: N-1 reduce-scatter steps, then N-1 allgather steps
        for i in range(N - 1):
            for b in range(N):
                u = us[(b - i) % N]
                ledger.move("phase2_rs", topo.rank(b, g), topo.rank((b + 1) % N, g), u.end - u.start)
                u = us[(b + 1 - i) % N]
                ledger.move("phase2_ag", topo.rank(b, g), topo.rank((b + 1) % N, g), u.end - u.start)


def _sentinel(dtype: str):
    # a value no reduction of the seeded inputs produces is not needed for
    # correctness: coverage is checked through the ownership maps (V4)
    return {"int32": np.int32(0), "float32": np.float32(0), "bfloat16": np.uint16(0)}[dtype]


# --------------------------------------------------------------------------
# plain definitions (pins for the simulation above)
# --------------------------------------------------------------------------
def brute_force_sum(xs, dtype: str) -> np.ndarray:
    """The plain definition, independent of the method's order: int32 ->
    exact int64 sum reduced mod 2^32 (R#9); fp -> float64 sum of the exactly
    widened inputs. Returns int32 or float64."""
    if dtype == "int32":
        s = np.zeros(len(xs[0]), np.int64)
        for x in xs:
            s += np.asarray(x, np.int64)
        return (s & 0xFFFFFFFF).astype(np.uint32).view(np.int32)
    s = np.zeros(len(xs[0]), np.float64)
    for x in xs:
        s += to_float64(x, dtype)
    return s


def abs_sum(xs, dtype: str) -> np.ndarray:
    s = np.zeros(len(xs[0]), np.float64)
    for x in xs:
        s += np.abs(to_float64(x, dtype))
    return s


def to_float64(x, dtype: str) -> np.ndarray:
    if dtype == "bfloat16":
        return (np.asarray(x, np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)
    return np.asarray(x).astype(np.float64)


TOLERANCE = {"float32": 1e-6, "bfloat16": 1e-2}  # north_star; R#10 (relative to sum|x|)
