"""Quick device timing of the emulated lane allreduce (dev tool, not the bench).

python tools/quick_time.py --layout 2x4 --k 1 --dtype float32 --mib 1024
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2508_13397_b200 as lane  # noqa: E402
from seeded_inputs import device as sdev  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layout", default="2x4")
    ap.add_argument("--k", type=int, default=1)
    ap.add_argument("--dtype", default="float32")
    ap.add_argument("--mib", type=float, default=1024)
    ap.add_argument("--iters", type=int, default=10)
    a = ap.parse_args()
    N, G = map(int, a.layout.split("x"))
    P = N * G
    tdt = {"int32": torch.int32, "float32": torch.float32, "bfloat16": torch.bfloat16}[a.dtype]
    isz = 2 if a.dtype == "bfloat16" else 4
    n = int(a.mib * (1 << 20)) // isz
    emu = lane.LaneEmulator(N, G, a.k, device=0)
    ins = [sdev.fill(torch.empty(n, dtype=tdt, device="cuda"), a.dtype, "signed", 42, p) for p in range(P)]
    outs = [torch.empty_like(t) for t in ins]
    for _ in range(3):
        emu.allreduce(outs, ins)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(a.iters):
        emu.allreduce(outs, ins)
    e.record()
    torch.cuda.synchronize()
    emu.check()
    ms = s.elapsed_time(e) / a.iters
    S = n * isz
    print(f"emulated {a.layout} k={a.k} {a.dtype} {S / 2**20:.0f} MiB/rank: {ms:.3f} ms  "
          f"plan={emu.plan(n, a.dtype)}  HBM-min(2PS)={2 * P * S / ms / 1e6:.0f} GB/s")


if __name__ == "__main__":
    main()
