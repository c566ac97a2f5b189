"""Host-side cost of one allreduce call (dev tool): the Python binding's
``comm.allreduce`` vs the bare C ABI call with pre-computed arguments vs a
plain torch kernel launch, median wall time per call over many calls
(the GPU work is tiny, so the host is the bottleneck being measured).

torchrun --nproc-per-node 2 tools/host_overhead.py
"""
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2508_13397_b200 as lane  # noqa: E402
from paper_2508_13397_b200 import _lib  # noqa: E402


def per_call_us(fn, n=2000):
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
    return statistics.median(ts) * 1e6


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    comm = lane.LaneComm(1, world, 1, rank=rank, device=local)
    x = torch.ones(1024, device="cuda")
    y = torch.empty_like(x)
    for _ in range(50):
        comm.allreduce(y, x)
    torch.cuda.synchronize()
    dist.barrier()
    lib = _lib.load()
    h = comm._comm
    sp = torch.cuda.current_stream().cuda_stream
    xp, yp = x.data_ptr(), y.data_ptr()
    res = {
        "binding comm.allreduce": per_call_us(lambda: comm.allreduce(y, x)),
        "C ABI lane_allreduce (pre-computed args)": per_call_us(lambda: lib.lane_allreduce(h, xp, yp, 1024, 1, 0, sp)),
        "torch.cuda.current_stream()": per_call_us(lambda: torch.cuda.current_stream()),
        "torch add_ (one kernel launch)": per_call_us(lambda: y.add_(x)),
    }
    dist.barrier()
    if rank == 0:
        for k, v in res.items():
            print(f"{k:45s} {v:7.2f} us", flush=True)
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
