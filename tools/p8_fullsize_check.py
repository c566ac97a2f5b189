"""P = 8 at BASELINE's full size through the multi-process path on a box with
fewer GPUs (dev tool; ranks spread rank % LANE_TEST_GPUS): the bench's own
launch configuration (registered buffers, default protocol and plan) for the
given layouts, then EVERY output element of every rank verified bit-exactly on
the device (bench.check_outputs). Correctness only: with several ranks per
GPU the kernels share the GPU, so no timing is reported.

LANE_TEST_GPUS=2 torchrun --nproc-per-node 8 --master-addr 127.0.0.1 tools/p8_fullsize_check.py \
    --layouts 2x4 4x2 8x1 --mib 1024 [--k 4] [--dtype bfloat16]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
import paper_2508_13397_b200 as lane  # noqa: E402
from seeded_inputs import device as sdev  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layouts", nargs="+", default=["2x4"])
    ap.add_argument("--mib", type=float, default=1024.0)
    ap.add_argument("--dtype", default="float32")
    ap.add_argument("--calls", type=int, default=2)
    ap.add_argument("--k", type=int, default=1)
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = rank % int(os.environ.get("LANE_TEST_GPUS", "1"))
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")
    os.environ.setdefault("LANE_TIMEOUT_MS", "120000")
    tdt = getattr(torch, a.dtype)
    n = int(a.mib * (1 << 20)) // tdt.itemsize
    bad = 0
    for lay in a.layouts:
        N, G = map(int, lay.split("x"))
        t0 = time.time()
        comm = lane.LaneComm(N, G, a.k, rank=rank, device=dev)
        inp = sdev.fill(torch.empty(n, dtype=tdt, device="cuda"), a.dtype, "signed", 42, rank)
        out = torch.empty_like(inp)
        comm.register(inp)
        comm.register(out)
        for _ in range(a.calls):
            comm.allreduce(out, inp)
        torch.cuda.synchronize()
        comm.check()
        chk = bench.check_outputs([out], N, G, a.dtype, n, 42)
        t = torch.tensor([0 if chk["verified"] else 1, chk["elements"] or 0], dtype=torch.int64)
        dist.all_reduce(t)
        bad += int(t[0])
        if rank == 0:
            print(f"p8_fullsize_check {lay} k={a.k} {a.dtype} {n * tdt.itemsize >> 20} MiB/rank protocol "
                  f"{comm.protocol(n, a.dtype)} plan {comm.plan(n, a.dtype)}: "
                  f"{'OK' if int(t[0]) == 0 else 'FAILED'} ({int(t[1])} elements verified, {chk['how']}) "
                  f"in {time.time() - t0:.1f}s", flush=True)
        dist.barrier()
        comm.close()
        del inp, out
        torch.cuda.empty_cache()
        dist.barrier()
    dist.destroy_process_group()
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
