"""CPU oracle for "Approach 2" of arXiv 2508.13397: on-node allreduce, then
off-node allreduce (a bullet of the commented-out draft of
§3 "Methods": "Approach 2: allreduce on node + allreduce off node").

TEST INFRASTRUCTURE ONLY (same rule as ``lane_oracle.py``).

Simulated step by step for P = N*G ranks (rank p = a*G + g, R#6), per
(round, k-slice, pipeline chunk) exactly as the lane method partitions the
message (``lane_oracle.partition``'s rounds / slices / chunks, R#2-R#4):

  S1 node RS   GPU (a,g) sums node part g (the remainder-first split of the
               chunk into G) over h = 0..G-1 ascending, ONE rounding -> T_a
  S2 node AG   every node member receives every part of T_a
  S3 lane RS   the chunk is split remainder-first into N lane parts V_b; GPU
               (a,g) sums V_a over the lane members b = 0..N-1 ascending, ONE
               rounding -> F (every lane g does this for the whole chunk)
  S4 lane AG   every lane member receives every V_b of F

Reading R#24: "allreduce" inside each stage is the direct reduce-scatter +
allgather of R#5, in the canonical order R#7. Each element is therefore
sum_b (sum_h x) with the same association and rounding points as the lane
method (R#7/R#8): the outputs are bit-identical to ``lane_allreduce``; what
differs is the traffic — the lane stage carries the whole buffer on every
lane, 2(G-1)/G*n on node plus 2(N-1)/N*n off node per rank.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .lane_oracle import ITEMSIZE, STORAGE, add, narrow, partition, split_remainder_first, widen


@dataclass
class Approach2Result:
    out: list
    sent: dict   # stage -> np.array[P] elements sent
    recv: dict


def approach2_allreduce(xs, N: int, G: int, k: int = 1, dtype: str = "float32",
                        chunk_granules: int | None = None,
                        round_granules: int | None = None) -> Approach2Result:
    P = N * G
    xs = [np.asarray(x, dtype=STORAGE[dtype]) for x in xs]
    if len(xs) != P:
        raise ValueError(f"need {P} input buffers, got {len(xs)}")
    n = len(xs[0])
    stages = ("node_rs", "node_ag", "lane_rs", "lane_ag")
    sent = {s: np.zeros(P, np.int64) for s in stages}
    recv = {s: np.zeros(P, np.int64) for s in stages}
    out = [np.zeros(n, STORAGE[dtype]) for _ in range(P)]

    def move(stage, src, dst, cnt):
        if src != dst:
            sent[stage][src] += cnt
            recv[stage][dst] += cnt

    # chunks (element ranges) from the lane method's partition: union of a chunk's units
    chunks = {}
    for u in partition(n, ITEMSIZE[dtype], N, G, k, chunk_granules, round_granules):
        key = (u.round, u.l, u.c)
        s, e = chunks.get(key, (u.part_start, u.part_end))
        chunks[key] = (min(s, u.part_start), max(e, u.part_end))
    q = 16 // ITEMSIZE[dtype]
    for (c0, c1) in chunks.values():
        g0, ng = c0 // q, -(-(c1 - c0) // q)  # chunk in granules (only the message's last may be partial)

        def el(gr):
            return min(c0 + gr * q, c1)

        # S1 + S2: node allreduce of the whole chunk, part by part
        T = [np.zeros(c1 - c0, STORAGE[dtype]) for _ in range(N)]
        for g, (p0, pl) in enumerate(split_remainder_first(ng, G)):
            s, e = el(p0), el(p0 + pl)
            for a in range(N):
                acc = widen(xs[a * G][s:e], dtype)
                for h in range(1, G):
                    acc = add(acc, widen(xs[a * G + h][s:e], dtype), dtype)
                T[a][s - c0:e - c0] = narrow(acc, dtype)
                for h in range(G):
                    move("node_rs", a * G + h, a * G + g, e - s)
                    move("node_ag", a * G + g, a * G + h, e - s)
        # S3 + S4: lane allreduce of the whole chunk on every lane g
        for b, (v0, vl) in enumerate(split_remainder_first(ng, N)):
            s, e = el(v0), el(v0 + vl)
            acc = widen(T[0][s - c0:e - c0], dtype)
            for bb in range(1, N):
                acc = add(acc, widen(T[bb][s - c0:e - c0], dtype), dtype)
            F = narrow(acc, dtype)
            for g in range(G):
                for bb in range(N):
                    move("lane_rs", bb * G + g, b * G + g, e - s)
                    move("lane_ag", b * G + g, bb * G + g, e - s)
                    out[bb * G + g][s:e] = F
    return Approach2Result(out, sent, recv)
