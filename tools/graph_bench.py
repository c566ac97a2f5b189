"""Eager calls vs the same calls replayed from a CUDA graph.

torchrun --nproc-per-node P tools/graph_bench.py --layout 2x2 --mib 1 4 16 [--out rows.jsonl]

For each size (a fresh comm, so its eager calls run with host epochs): 20
back-to-back allreduce calls timed eagerly (CUDA events on the stream, max
over ranks, median of 3), then the same 20 calls captured into one CUDA graph
and replayed (device-side epochs); busbw for both, NVML clocks,
and the WHOLE output buffer of every rank verified bit-exactly on the device
after the last replay (bench.check_outputs).
"""
import json
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
    ap.add_argument("--out", default=None, help="append one JSON row per size (rank 0)")
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
        clk = bench.Clocks(list(range(world))) if rank == 0 else None
        if clk:
            clk.__enter__()
        cur = torch.cuda.current_stream()
        eager = lambda: [comm.allreduce(out, inp) for _ in range(a.calls)]  # noqa: E731
        me = bench.timed_repeats(eager, 1, 2, cur, dist, 3)
        s.wait_stream(cur)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            g.capture_begin()
            for _ in range(a.calls):
                comm.allreduce(out, inp)
            g.capture_end()
        cur.wait_stream(s)
        mg = bench.timed_repeats(g.replay, 1, 2, cur, dist, 3)
        if clk:
            clk.__exit__()
        comm.check()
        chk = bench.check_outputs([out], N, G, "float32", n, 42)
        t = torch.tensor([0.0 if chk["verified"] else 1.0], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        S = n * 4
        ms_e, ms_g = me[0] / a.calls, mg[0] / a.calls
        row = {"layout": a.layout, "bytes": S, "protocol": comm.protocol(n, "float32"), "calls": a.calls,
               "eager_us": round(ms_e * 1e3, 2), "graph_us": round(ms_g * 1e3, 2),
               "eager_busbw": round(bench.busbw(S, world, ms_e), 2), "graph_busbw": round(bench.busbw(S, world, ms_g), 2),
               "verified": t.item() == 0, "verified_how": chk["how"] + " (after the last replay)",
               "clocks": clk.summary() if clk else None}
        if rank == 0:
            print(json.dumps(row), flush=True)
            if a.out:
                with open(a.out, "a") as f:
                    f.write(json.dumps(row) + "\n")
        del g
        torch.cuda.synchronize()
        dist.barrier()
        comm.close()
        dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
