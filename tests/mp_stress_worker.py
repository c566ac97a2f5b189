"""Stress (multi-GPU): thousands of back-to-back allreduces on one comm,
alternating the LL, LL128 and simple protocols, sizes across their thresholds and
the bulk-store threshold, registered and unregistered buffers, in-place and
out-of-place — every call checked exactly (int32: the expected sum is a
closed form, computed on the device with plain torch ops). Looks for rare
races in epoch / parity-set / scratch reuse that a few calls would not hit.

    torchrun --nproc-per-node P --master-addr 127.0.0.1 tests/mp_stress_worker.py [--iters N]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2508_13397_b200 as lane  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=2000)
    ap.add_argument("--layout", default=None)
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    os.environ.setdefault("LANE_TIMEOUT_MS", "10000")
    N, G = map(int, a.layout.split("x")) if a.layout else (2, world // 2) if world % 2 == 0 else (world, 1)
    comm = lane.LaneComm(N, G, 2, rank=rank, device=local)
    nmax = (24 << 20) // 4  # 24 MiB of int32
    rin = torch.empty(nmax, dtype=torch.int32, device="cuda")
    rout = torch.empty_like(rin)
    comm.register(rin)
    comm.register(rout)
    # LL (<= 1 MiB), LL128 (1-16 MiB), simple, simple with bulk stores (>= 16 MiB)
    sizes = [1, 1000, 4099, 1 << 18, (3 << 18) + 5, (1 << 21) + 3, (1 << 22) - 1, (2 << 20) + 17, (5 << 20) + 1, nmax]
    g = torch.Generator().manual_seed(1234)  # same sequence on every rank
    bad = 0
    t0 = time.time()
    for it in range(a.iters):
        n = sizes[int(torch.randint(len(sizes), (1,), generator=g))]
        mode = int(torch.randint(4, (1,), generator=g))  # registered? in place?
        registered, inplace = mode & 1, mode & 2
        idx = torch.arange(n, device="cuda", dtype=torch.int64)
        base = (idx * 7 + it) % (1 << 20)
        inp = rin[:n] if registered else torch.empty(n, dtype=torch.int32, device="cuda")
        inp.copy_((base + 13 * rank).to(torch.int32))
        out = inp if inplace else (rout[:n] if registered else torch.empty_like(inp))
        comm.allreduce(out, inp)
        want = (base * world + 13 * (world * (world - 1) // 2)).to(torch.int32)
        if not torch.equal(out, want):
            bad += 1
            if bad < 5:
                print(f"rank {rank} it {it} n={n} mode={mode} proto={comm.protocol(n, 'int32')}: MISMATCH "
                      f"({int((out != want).sum())} elements)", flush=True)
    torch.cuda.synchronize()
    comm.check()
    t = torch.tensor([bad])
    dist.all_reduce(t)
    if rank == 0:
        print(f"mp_stress_worker P={world} {N}x{G}: {'OK' if t.item() == 0 else 'FAILED'} ({t.item()} bad calls of "
              f"{a.iters}) in {time.time() - t0:.1f}s", flush=True)
    comm.close()
    dist.destroy_process_group()
    sys.exit(1 if t.item() else 0)


if __name__ == "__main__":
    main()
