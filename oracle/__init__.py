"""CPU oracle for the multi-lane allreduce (arXiv 2508.13397, Alg. 2 + §3.1.2).

TEST INFRASTRUCTURE ONLY — not part of the product. Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it. It shares no code with
``paper_2508_13397_b200/`` (the CUDA path) and never imports it.

Parity pinning status:
  topology / partition / ledger ....... pinned (closed forms, SPEC examples, enumeration)
  int32 results ....................... pinned (plain definition: exact sum mod 2^32)
  fp32 / bf16 results (value) ......... pinned (float64 brute force within the error bound)
  fp32 / bf16 results (exact bits) .... pinned by the canonical-order fixture
                                        tests/golden/canonical_order.txt (reading R#7/R#8)
"""
from .lane_oracle import (  # noqa: F401
    GRANULE_BYTES,
    ITEMSIZE,
    TOLERANCE,
    Ledger,
    OracleResult,
    Topology,
    Unit,
    abs_sum,
    bf16_round_nearest_even,
    brute_force_sum,
    lane_allreduce,
    partition,
    split_remainder_first,
    to_float64,
)
from .ring_oracle import RingResult, ring_allreduce, ring_chunks  # noqa: F401,E402
from .approach2_oracle import Approach2Result, approach2_allreduce  # noqa: F401,E402
