"""Watchdog check (multi-GPU, P = 2): rank 0 calls an allreduce that rank 1
never joins. Rank 0's kernel must give up after LANE_TIMEOUT_MS (the device
watchdog, include/lane_allreduce.h LANE_ERR_TIMEOUT) instead of hanging, the
comm must then report LANE_ERR_TIMEOUT on check() and on the next call, and
both ranks must shut down cleanly. One case per signalling protocol. Then
the call-signature cases (mismatch_cases): ranks that disagree on a call end
with LANE_ERR_MISMATCH instead of a timeout or wrong data.

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


def mismatch_cases(rank, world, local):
    """Ranks that disagree on a simple-protocol call (a buffer registered on
    one rank only; different offsets into the registrations; different
    counts) must all stop in the start handshake with LANE_ERR_MISMATCH (-7),
    promptly (the watchdog is 20 s here), and leave the recvbufs untouched."""
    bad = 0
    os.environ["LANE_TIMEOUT_MS"] = "20000"
    os.environ["LANE_PROTO"] = "simple"
    n = 1 << 20
    for case in ("registered_on_one_rank", "offsets", "count"):
        comm = lane.LaneComm(1, world, 1, rank=rank, device=local)
        rin = torch.ones(n + 64, device="cuda")
        rout = torch.empty_like(rin)
        comm.register(rin)
        comm.register(rout)
        if case == "registered_on_one_rank":
            x, y = (rin[:n], rout[:n]) if rank == 0 else (torch.ones(n, device="cuda"), torch.empty(n, device="cuda"))
        elif case == "offsets":
            o = 0 if rank == 0 else 16
            x, y = rin[o:o + n], rout[o:o + n]
        else:
            m = n if rank == 0 else n + 4
            x, y = rin[:m], rout[:m]
        y.view(torch.int32).fill_(-1)
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.time()
        comm.allreduce(y, x)
        torch.cuda.synchronize()
        dt = time.time() - t0
        try:
            comm.check()
            print(f"rank {rank} mismatch/{case}: not reported", flush=True)
            bad += 1
        except lane.LaneError as e:
            if e.code != -7:
                print(f"rank {rank} mismatch/{case}: code {e.code}", flush=True)
                bad += 1
        if not bool((y.view(torch.int32) == -1).all()):
            print(f"rank {rank} mismatch/{case}: recvbuf written", flush=True)
            bad += 1
        if dt > 5:
            print(f"rank {rank} mismatch/{case}: took {dt:.1f}s", flush=True)
            bad += 1
        print(f"rank {rank} mismatch/{case}: LANE_ERR_MISMATCH after {dt:.3f}s", flush=True)
        dist.barrier()
        comm.close()
        dist.barrier()
    return bad


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    # LANE_TEST_DEVICE=d puts every rank on GPU d (ranks sharing one GPU: the 1-GPU tier);
    # LANE_TEST_GPUS=g spreads the ranks over g GPUs (rank % g; P = 8 on fewer GPUs)
    if "LANE_TEST_GPUS" in os.environ:
        local = rank % int(os.environ["LANE_TEST_GPUS"])
    else:
        local = int(os.environ.get("LANE_TEST_DEVICE", os.environ.get("LOCAL_RANK", rank)))
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
    bad += mismatch_cases(rank, world, local)
    t = torch.tensor([bad])
    dist.all_reduce(t)
    if rank == 0:
        print(f"mp_timeout_worker: {'OK' if t.item() == 0 else 'FAILED'}", flush=True)
    dist.destroy_process_group()
    sys.exit(1 if t.item() else 0)


if __name__ == "__main__":
    main()
