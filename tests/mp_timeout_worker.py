"""Watchdog check (multi-GPU, P = 2): rank 0 calls an allreduce that rank 1
never joins. Rank 0's kernel must give up after LANE_TIMEOUT_MS (the device
watchdog, include/lane_allreduce.h LANE_ERR_TIMEOUT) instead of hanging, the
comm must then report LANE_ERR_TIMEOUT on check() and on the next call, and
both ranks must shut down cleanly. One case per signalling protocol.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tests/mp_timeout_worker.py
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2508_13397_b200 as lane  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    os.environ["LANE_TIMEOUT_MS"] = "1500"
    bad = 0
    for proto, n in (("simple", 1 << 20), ("ll", 4099), ("ll128", 1 << 20)):
        os.environ["LANE_PROTO"] = proto
        comm = lane.LaneComm(1, world, 1, rank=rank, device=local)
        x = torch.ones(n, device="cuda")
        y = torch.empty_like(x)
        dist.barrier()
        if rank == 0:
            t0 = time.time()
            comm.allreduce(y, x)
            torch.cuda.synchronize()  # returns only because the watchdog fired
            dt = time.time() - t0
            try:
                comm.check()
                print(f"rank 0 {proto}: no timeout reported", flush=True)
                bad += 1
            except lane.LaneError as e:
                if e.code != -5:
                    bad += 1
            try:
                comm.allreduce(y, x)
                print(f"rank 0 {proto}: call after a timeout was accepted", flush=True)
                bad += 1
            except lane.LaneError as e:
                if e.code != -5:
                    bad += 1
            print(f"rank 0 {proto}: watchdog fired after {dt:.2f}s", flush=True)
            if dt > 30:
                bad += 1
        dist.barrier()
        comm.close()
        dist.barrier()
    t = torch.tensor([bad])
    dist.all_reduce(t)
    if rank == 0:
        print(f"mp_timeout_worker: {'OK' if t.item() == 0 else 'FAILED'}", flush=True)
    dist.destroy_process_group()
    sys.exit(1 if t.item() else 0)


if __name__ == "__main__":
    main()
