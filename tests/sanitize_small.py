"""Small emulated runs of every kernel for compute-sanitizer (test harness, so it
lives under tests/ — it checks against oracle/):
simple (TMA, LSU-store and bulk-store), LL, LL128, ring (LL, LL128) and approach 2,
2x2 and 1x3 layouts, counts with ragged tails. Exits non-zero on a parity
failure. compute-sanitizer --tool memcheck python tests/sanitize_small.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("LANE_TIMEOUT_MS", "300000")
os.environ.setdefault("LANE_ROUND_BYTES", str(1 << 20))
os.environ.setdefault("LANE_LL_MAX_BYTES", str(256 << 10))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import seeded_inputs as si  # noqa: E402
import paper_2508_13397_b200 as lane  # noqa: E402
from tests.gpu_util import bits, to_device, to_numpy  # noqa: E402


def run(N, G, k, n, proto, algo, store="lsu"):
    os.environ["LANE_PROTO"] = proto
    os.environ["LANE_STORE"] = store
    e = lane.LaneEmulator(N, G, k, device=0)
    xs = si.generate_all("float32", "signed", 5 + n, N * G, n)
    ins = [to_device(x, "float32", "cuda:0") for x in xs]
    outs = [torch.zeros_like(t) for t in ins]
    getattr(e, {"lane": "allreduce", "ring": "allreduce_ring", "a2": "allreduce_approach2"}[algo])(outs, ins)
    torch.cuda.synchronize()
    e.check()
    if algo == "ring":
        pl = e.plan(n, "float32", algorithm="ring")
        ref = oracle.ring_allreduce(xs, k, "float32", pl["chunk_granules"], pl["round_granules"]).out[0]
    else:
        ref = oracle.lane_allreduce(xs, N, G, k, "float32").out[0]
    ok = all(np.array_equal(bits(to_numpy(o, "float32")), bits(ref)) for o in outs)
    e.close()
    print(f"{N}x{G} k={k} n={n} {proto} {algo} {store}: {'ok' if ok else 'MISMATCH'}", flush=True)
    return ok


def main():
    ok = True
    for (N, G) in ((2, 2), (1, 3)):
        for n in (4099, 70001):
            ok &= run(N, G, 2, n, "simple", "lane", "lsu")
            ok &= run(N, G, 2, n, "simple", "lane", "bulk")
            ok &= run(N, G, 2, n, "ll", "lane")
            ok &= run(N, G, 2, n, "ll", "ring")
            ok &= run(N, G, 2, n, "ll", "a2")
            ok &= run(N, G, 2, n, "ll128", "lane")
            ok &= run(N, G, 2, n, "ll128", "ring")
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
