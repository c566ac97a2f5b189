"""Stress (multi-GPU): thousands of back-to-back allreduces on one comm per
virtual layout, alternating the LL, LL128 and simple protocols, sizes across
their thresholds and the bulk-store threshold, int32 / fp32 / bf16, registered
and unregistered buffers, in-place and out-of-place — every call checked
bit-exactly on the device against the canonical-order sum (DESIGN R#7/R#8;
bench.canonical_lane_sum_torch, pinned to the oracle by the CPU tests) of the
P seeded inputs regenerated on the device. fp32 / bf16 matter here: an int32
closed form cannot see a torn LL128 line whose data happen to match (R#25).
Looks for rare races in epoch / parity-set / scratch reuse that a few calls
would not hit.

    torchrun --nproc-per-node P --master-addr 127.0.0.1 tests/mp_stress_worker.py [--iters N] [--layouts all|NxG]
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

TDT = {"int32": torch.int32, "float32": torch.float32, "bfloat16": torch.bfloat16}


def stress(N, G, iters, rank, world, local):
    comm = lane.LaneComm(N, G, 2, rank=rank, device=local)
    nbytes = 24 << 20
    rin = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    rout = torch.empty_like(rin)
    comm.register(rin)
    comm.register(rout)
    # bytes per rank: LL (<= 1 MiB), LL128 (1-16 MiB), simple, simple with bulk stores (>= 16 MiB)
    sizes = [4, 4000, 16396, 1 << 20, (3 << 20) + 20, (8 << 20) + 12, (16 << 20) - 4, (9 << 20) + 68,
             (20 << 20) + 4, nbytes]
    g = torch.Generator().manual_seed(1234 + N)  # same sequence on every rank
    bad = 0
    for it in range(iters):
        nb = sizes[int(torch.randint(len(sizes), (1,), generator=g))]
        dtype = ["int32", "float32", "bfloat16"][int(torch.randint(3, (1,), generator=g))]
        mode = int(torch.randint(4, (1,), generator=g))  # registered? in place?
        registered, inplace = mode & 1, mode & 2
        tdt = TDT[dtype]
        n = nb // (2 if dtype == "bfloat16" else 4)
        seed = 5000 + it
        dist_ = "full" if dtype == "int32" else "signed"
        inp = rin[:n * tdt.itemsize].view(tdt) if registered else torch.empty(n, dtype=tdt, device="cuda")
        sdev.fill(inp, dtype, dist_, seed, rank)
        out = inp if inplace else (rout[:n * tdt.itemsize].view(tdt) if registered else torch.empty_like(inp))
        comm.allreduce(out, inp)
        xs = [sdev.fill(torch.empty(n, dtype=tdt, device="cuda"), dtype, dist_, seed, p) for p in range(N * G)]
        want = bench.canonical_lane_sum_torch(xs, N, G, dtype)
        if not torch.equal(bench._bitview(out), bench._bitview(want)):
            bad += 1
            if bad < 5:
                print(f"rank {rank} {N}x{G} it {it} {dtype} n={n} mode={mode} proto={comm.protocol(n, dtype)}: "
                      f"MISMATCH ({int((bench._bitview(out) != bench._bitview(want)).sum())} elements)", flush=True)
    torch.cuda.synchronize()
    comm.check()
    dist.barrier()
    comm.close()
    dist.barrier()
    return bad


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=2000, help="calls per layout")
    ap.add_argument("--layouts", default="default", help="'all', 'default' (2 x P/2) or NxG")
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    # LANE_TEST_DEVICE=d puts every rank on GPU d (ranks sharing one GPU: the 1-GPU tier);
    # LANE_TEST_GPUS=g spreads the ranks over g GPUs (rank % g; P = 8 on fewer GPUs)
    if "LANE_TEST_GPUS" in os.environ:
        local = rank % int(os.environ["LANE_TEST_GPUS"])
    else:
        local = int(os.environ.get("LANE_TEST_DEVICE", os.environ.get("LOCAL_RANK", rank)))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    os.environ.setdefault("LANE_TIMEOUT_MS", "10000")
    if a.layouts == "all":
        layouts = [(N, world // N) for N in range(1, world + 1) if world % N == 0]
    elif a.layouts == "default":
        layouts = [(2, world // 2) if world % 2 == 0 else (world, 1)]
    else:
        layouts = [tuple(map(int, a.layouts.split("x")))]
    total = 0
    for N, G in layouts:
        t0 = time.time()
        bad = stress(N, G, a.iters, rank, world, local)
        t = torch.tensor([bad])
        dist.all_reduce(t)
        total += t.item()
        if rank == 0:
            print(f"mp_stress_worker P={world} {N}x{G}: {'OK' if t.item() == 0 else 'FAILED'} ({t.item()} bad calls "
                  f"of {a.iters}, int32/fp32/bf16 bit-exact) in {time.time() - t0:.1f}s", flush=True)
    dist.destroy_process_group()
    sys.exit(1 if total else 0)


if __name__ == "__main__":
    main()
