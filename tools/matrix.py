"""BASELINE configs[4] matrix in ONE torchrun job (dev/measurement tool): every
virtual layout N x G with N*G == world, k in {1,2,4,8}, int32 and fp32 (and
bf16 with --bf16), one message size (default 1 GiB per rank), plus NCCL ring
and the paper's multi-PPG CCL variant (--ppg communicators) per dtype.
Device time (CUDA events), max over ranks. Every cell: --repeats timed runs (median / min / max) with the clock record
(nvidia-smi / NVML: SM clock, throttle reasons) taken during them, and the
whole output buffer verified bit-exactly on the device (bench.check_outputs).
One JSON object per cell on rank 0.

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
    ap.add_argument("--repeats", type=int, default=3)
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

    def cell(fn):
        """a.repeats timed runs of a.iters calls (max over ranks each) with the
        nvidia-smi / NVML clock record of the cell (rank 0 samples all GPUs)."""
        clk = bench.Clocks(list(range(world))) if rank == 0 else None
        if clk:
            clk.__enter__()
        med, lo, hi = bench.timed_repeats(fn, a.iters, 3, stream, dist, a.repeats)
        if clk:
            clk.__exit__()
        return med, lo, hi, (clk.summary() if clk else None)

    def times(S, med, lo, hi, clocks):
        d = {"bytes": S, "ms": round(med, 4), "ms_min": round(lo, 4), "ms_max": round(hi, 4),
             "busbw": round(bench.busbw(S, world, med), 2), "busbw_min": round(bench.busbw(S, world, hi), 2),
             "busbw_max": round(bench.busbw(S, world, lo), 2), "repeats": a.repeats, "iters": a.iters}
        if clocks:
            d["clocks"] = clocks
        return d

    for dtype in a.dtypes:
        isz = bench.itemsize(dtype)
        n = int(a.mib * (1 << 20)) // isz
        S = n * isz
        tdt = getattr(torch, dtype)
        rin = torch.empty(n, dtype=tdt, device="cuda")
        rout = torch.empty_like(rin)
        sdev.fill(rin, dtype, "signed", 42, rank)
        buf = rin.clone()
        emit(dict({"impl": "nccl_ring", "P": world, "dtype": dtype, "algo": os.environ.get("NCCL_ALGO")},
                  **times(S, *cell(lambda: dist.all_reduce(buf)))))
        if ppg:
            emit(dict({"impl": f"nccl_ring_x{a.ppg}ppg", "P": world, "dtype": dtype},
                      **times(S, *cell(lambda: ppg.run(buf, dist)))))
        del buf
        for N, G in layouts:
            for k in a.ks:
                comm = lane.LaneComm(N, G, k, rank=rank, device=local)
                comm.register(rin)
                comm.register(rout)
                med, lo, hi, clocks = cell(lambda: comm.allreduce(rout, rin))
                comm.check()
                chk = bench.check_outputs([rout], N, G, dtype, n, 42)
                t = torch.tensor([0.0 if chk["verified"] else 1.0], dtype=torch.float64)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                row = {"impl": "lane", "P": world, "layout": f"{N}x{G}", "k": k, "dtype": dtype,
                       "verified": t[0].item() == 0, "verified_how": chk["how"],
                       "protocol": comm.protocol(n, dtype), "plan": comm.plan(n, dtype)}
                row.update(times(S, med, lo, hi, clocks))
                row["frac_of_770"] = round(row["busbw"] / 770.0, 4)
                emit(row)
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
