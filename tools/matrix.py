"""BASELINE configs[4] matrix in ONE torchrun job (dev/measurement tool): every
virtual layout N x G with N*G == world, k in {1,2,4,8}, int32 and fp32 (and
bf16 with --bf16), one message size (default 1 GiB per rank), plus NCCL ring
and the paper's multi-PPG CCL variant (--ppg communicators) per dtype.
Device time (CUDA events), max over ranks; every lane cell verified on
sampled elements against the oracle. One JSON object per cell on rank 0.

torchrun --nproc-per-node 4 --master-addr 127.0.0.1 tools/matrix.py --out gpurun_out/m4.jsonl
"""
import argparse
import json
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
    ap.add_argument("--mib", type=float, default=1024)
    ap.add_argument("--ks", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--dtypes", nargs="+", default=["float32", "int32"])
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--ppg", type=int, default=4)
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("cpu:gloo,cuda:nccl")
    stream = torch.cuda.current_stream()
    layouts = [(N, world // N) for N in range(1, world + 1) if world % N == 0]
    ppg = bench.NcclPPG(a.ppg, dist) if a.ppg > 1 else None
    rows = []

    def emit(row):
        rows.append(row)
        if rank == 0:
            print(json.dumps(row), flush=True)

    for dtype in a.dtypes:
        isz = bench.itemsize(dtype)
        n = int(a.mib * (1 << 20)) // isz
        S = n * isz
        tdt = getattr(torch, dtype)
        rin = torch.empty(n, dtype=tdt, device="cuda")
        rout = torch.empty_like(rin)
        sdev.fill(rin, dtype, "signed", 42, rank)
        buf = rin.clone()
        ms = bench.device_time_ms(lambda: dist.all_reduce(buf), a.iters, 3, stream, dist.barrier)
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        emit({"impl": "nccl_ring", "P": world, "dtype": dtype, "bytes": S, "ms": round(t.item(), 4),
              "busbw": round(bench.busbw(S, world, t.item()), 2), "algo": os.environ.get("NCCL_ALGO")})
        if ppg:
            ms = bench.device_time_ms(lambda: ppg.run(buf, dist), a.iters, 3, stream, dist.barrier)
            t = torch.tensor([ms], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            emit({"impl": f"nccl_ring_x{a.ppg}ppg", "P": world, "dtype": dtype, "bytes": S, "ms": round(t.item(), 4),
                  "busbw": round(bench.busbw(S, world, t.item()), 2)})
        del buf
        for N, G in layouts:
            for k in a.ks:
                comm = lane.LaneComm(N, G, k, rank=rank, device=local)
                comm.register(rin)
                comm.register(rout)
                ms = bench.device_time_ms(lambda: comm.allreduce(rout, rin), a.iters, 3, stream, dist.barrier)
                ok = bench.sample_check([rout], N, G, dtype, n, 42, [rank])
                t = torch.tensor([ms, 0.0 if ok else 1.0], dtype=torch.float64)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                bw = bench.busbw(S, world, t[0].item())
                emit({"impl": "lane", "P": world, "layout": f"{N}x{G}", "k": k, "dtype": dtype, "bytes": S,
                      "ms": round(t[0].item(), 4), "busbw": round(bw, 2), "frac_of_770": round(bw / 770.0, 4),
                      "verified": t[1].item() == 0, "protocol": comm.protocol(n, dtype), "plan": comm.plan(n, dtype)})
                torch.cuda.synchronize()
                dist.barrier()
                comm.close()
                dist.barrier()
        del rin, rout
        torch.cuda.empty_cache()
    if rank == 0:
        with open(a.out, "a") as f:
            for r in rows:
                f.write(json.dumps(r) + "\n")
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
