"""Eager calls vs the same calls replayed from a CUDA graph (dev tool).

torchrun --nproc-per-node P tools/graph_bench.py --layout 2x2 --mib 0.25 1 4 16

For each size: 20 back-to-back allreduce calls timed eagerly (CUDA events on
the stream, max over ranks), then the same 20 calls captured into one CUDA
graph and replayed (device-side epochs), busbw for both; the last
replay's output is checked on sampled elements.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
import paper_2508_13397_b200 as lane  # noqa: E402
from seeded_inputs import device as sdev  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layout", default="2x2")
    ap.add_argument("--mib", type=float, nargs="+", default=[0.25, 1, 4, 16])
    ap.add_argument("--calls", type=int, default=20)
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    N, G = map(int, a.layout.split("x"))
    nmax = int(max(a.mib) * (1 << 20)) // 4
    rin = torch.empty(nmax, device="cuda")
    rout = torch.empty_like(rin)
    s = torch.cuda.Stream()
    for mib in a.mib:
        # a fresh comm per size: its eager calls run with host epochs, before its first capture
        comm = lane.LaneComm(N, G, 1, rank=rank, device=local)
        comm.register(rin)
        comm.register(rout)
        n = int(mib * (1 << 20)) // 4
        inp, out = rin[:n], rout[:n]
        sdev.fill(inp, "float32", "signed", 42, rank)
        torch.cuda.synchronize()
        dist.barrier()
        ms_e = bench.device_time_ms(lambda: [comm.allreduce(out, inp) for _ in range(a.calls)], 3, 2,
                                    torch.cuda.current_stream(), dist.barrier) / a.calls
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            g.capture_begin()
            for _ in range(a.calls):
                comm.allreduce(out, inp)
            g.capture_end()
        torch.cuda.current_stream().wait_stream(s)
        ms_g = bench.device_time_ms(g.replay, 3, 2, torch.cuda.current_stream(), dist.barrier) / a.calls
        comm.check()
        ok = bench.sample_check([out], N, G, "float32", n, 42, [rank])
        t = torch.tensor([ms_e, ms_g, 0.0 if ok else 1.0], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        S = n * 4
        if rank == 0:
            print(f"{a.layout} {mib:g} MiB proto={comm.protocol(n, 'float32')}: eager {t[0].item() * 1e3:.1f} us "
                  f"({bench.busbw(S, world, t[0].item()):.0f} GB/s)  graph {t[1].item() * 1e3:.1f} us "
                  f"({bench.busbw(S, world, t[1].item()):.0f} GB/s)  verified={t[2].item() == 0}", flush=True)
        del g
        torch.cuda.synchronize()
        dist.barrier()
        comm.close()
        dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
