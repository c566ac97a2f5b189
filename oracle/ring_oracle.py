"""CPU oracle for the ring allreduce of arXiv 2508.13397, Algorithm 1.

TEST INFRASTRUCTURE ONLY (same rule as ``lane_oracle.py``: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may import it; it
imports nothing from the product path).

Algorithm 1 ``ring_allreduce`` (P L150-206, §2.1) is the "standard" large
allreduce the paper compares the multi-lane algorithm with
(fig:std_vs_lane, fig:full_mpi_comparison, P L393-401); applied per k-slice
it is the paper's "standard approach" with multiple processes per GPU
(§3.1.1, P L335-349: every process l_r allreduces its own s/PPG slice).

Simulated literally, per k-slice, on n = P ranks:

  chunks     c_chunk = c_buf / n with counts c_on_chunk and displacements D
             (P L156-171); the remainder the paper drops is spread
             remainder-first over 16-byte granules (reading R#2).
  RS loop    for i in [0, n-1) (exclusive bound, R#1): rank r sends chunk sp
             (of buf_sendfrom: sendbuf at i = 0, recvbuf after) to r+1 and
             receives chunk rp from r-1, reducing it with its own sendbuf
             chunk into recvbuf (MPI_Reduce, P L177-181); sp = r, rp = r-1
             initially, both decrement mod n each step (P L183-187).
  AG loop    sp = r+1, rp = r; n-1 exchange steps of recvbuf chunks
             (MPI_Isend/Irecv/Waitall, P L192-203).

Arithmetic: each hop is ONE binary reduction in the buffer's type, as an
MPI_Reduce on that buffer performs it: int32 wrap (R#9), fp32 RNE, bf16
widened exactly to fp32, added, rounded to nearest-even once per hop (reading
R#11: per-hop rounding — the ring's own arithmetic; IEEE addition is
commutative, so the operand order inside a hop does not matter). Chunk c is
therefore ((x_c + x_{c+1}) + x_{c+2}) + ... + x_{c-1}, ending on rank c-1.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .lane_oracle import GRANULE_BYTES, ITEMSIZE, STORAGE, narrow, split_remainder_first, widen


@dataclass
class RingResult:
    out: list              # per-rank outputs (storage dtype)
    sent: np.ndarray       # elements sent per rank (RS + AG)
    recv: np.ndarray       # elements received per rank
    owner: np.ndarray      # [n] rank that completed the reduction of element i
    messages: np.ndarray   # messages sent per rank


def ring_chunks(n: int, itemsize: int, P: int, k: int = 1, chunk_granules: int | None = None,
                round_granules: int | None = None) -> list[list[tuple[int, int]]]:
    """The independent rings of a message: for every (round, k-slice, pipeline
    chunk), the element ranges [start, end) of its P ring chunks. Rounds are
    consecutive pieces of ``round_granules`` 16-byte granules, slices the
    remainder-first split of a round into k (R#3), pipeline chunks
    consecutive pieces of ``chunk_granules`` of a slice (R#21: Alg. 1 runs on
    every pipeline chunk; None = the whole slice, the paper's one-shot
    form), ring chunks the remainder-first split of a pipeline chunk into P
    (R#2); clipped at n. Same hierarchy as ``lane_oracle.partition``."""
    q = GRANULE_BYTES // itemsize
    ng = -(-n // q)
    out = []
    if ng == 0:
        return out
    rg = round_granules or ng
    for r0 in range(0, ng, rg):
        rlen = min(rg, ng - r0)
        for s0, slen in split_remainder_first(rlen, k):
            cg = chunk_granules or max(slen, 1)
            for c0 in range(0, slen, cg):
                clen = min(cg, slen - c0)
                base = r0 + s0 + c0
                out.append([(min((base + p0) * q, n), min((base + p0 + pl) * q, n))
                            for p0, pl in split_remainder_first(clen, P)])
    return out


def _hop(incoming: np.ndarray, own: np.ndarray, dtype: str) -> np.ndarray:
    """One MPI_Reduce hop in the buffer type."""
    with np.errstate(over="ignore"):
        return narrow(widen(incoming, dtype) + widen(own, dtype), dtype)


def ring_allreduce(xs, k: int = 1, dtype: str = "float32", chunk_granules: int | None = None,
                   round_granules: int | None = None) -> RingResult:
    """Simulate Alg. 1 on every independent ring (k-slice, or pipeline chunk
    of a slice, see ``ring_chunks``) of the P = len(xs) ranks' buffers."""
    P = len(xs)
    xs = [np.asarray(x, dtype=STORAGE[dtype]) for x in xs]
    n = len(xs[0])
    if any(len(x) != n for x in xs):
        raise ValueError("all ranks must pass the same count (P L341 collective semantics)")
    recv = [np.zeros(n, STORAGE[dtype]) for _ in range(P)]
    sent = np.zeros(P, np.int64)
    got = np.zeros(P, np.int64)
    msgs = np.zeros(P, np.int64)
    owner = np.full(n, -1, np.int64)
    if P == 1:
        return RingResult([xs[0].copy()], sent, got, np.zeros(n, np.int64), msgs)
    for D in ring_chunks(n, ITEMSIZE[dtype], P, k, chunk_granules, round_granules):
        # reduce-scatter loop (P L175-188)
        sp = list(range(P))
        rp = [(r - 1) % P for r in range(P)]
        sendfrom = [xs[r] for r in range(P)]
        for _ in range(P - 1):
            # every rank posts its message, then every rank reduces what it got
            msg = []
            for r in range(P):
                s, e = D[sp[r]]
                msg.append(sendfrom[r][s:e].copy())
                sent[r] += e - s
                msgs[r] += 1
            for r in range(P):
                s, e = D[rp[r]]
                incoming = msg[(r - 1) % P]  # chunk rp[r] of rank r-1 (its sp == my rp)
                recv[r][s:e] = _hop(incoming, xs[r][s:e], dtype)
                got[r] += e - s
            sp = [(v - 1) % P for v in sp]
            rp = [(v - 1) % P for v in rp]
            sendfrom = recv
        for r in range(P):  # rank r completed chunk r+1 (its last rp)
            s, e = D[(r + 1) % P]
            owner[s:e] = r
        # allgather loop (P L190-203)
        sp = [(r + 1) % P for r in range(P)]
        rp = list(range(P))
        for _ in range(P - 1):
            msg = []
            for r in range(P):
                s, e = D[sp[r]]
                msg.append(recv[r][s:e].copy())
                sent[r] += e - s
                msgs[r] += 1
            for r in range(P):
                s, e = D[rp[r]]
                recv[r][s:e] = msg[(r - 1) % P]
                got[r] += e - s
            sp = [(v - 1) % P for v in sp]
            rp = [(v - 1) % P for v in rp]
    return RingResult(recv, sent, got, owner, msgs)
