"""Tune the multi-GPU lane allreduce over LANE_* settings in ONE torchrun job
(dev tool; every config re-creates the comm, since most knobs are read at
init). Prints busbw (GB/s, max-over-ranks device time) per config and size,
with every cell verified on sampled elements against the oracle.

torchrun --nproc-per-node 4 tools/tune_mid.py --layout 2x2 --mib 8 16 32 \
    --cfg "" "LANE_CTAS_TOTAL=64" "LANE_PROTO=simple,LANE_CHUNKS_PER_CTA=1"
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
    ap.add_argument("--k", type=int, default=1)
    ap.add_argument("--dtype", default="float32")
    ap.add_argument("--mib", type=float, nargs="+", default=[8, 16, 32])
    ap.add_argument("--cfg", nargs="+", default=[""])
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--nccl", action="store_true")
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("cpu:gloo,cuda:nccl")
    N, G = map(int, a.layout.split("x"))
    isz = 2 if a.dtype == "bfloat16" else 4
    tdt = getattr(torch, a.dtype)
    nmax = int(max(a.mib) * (1 << 20)) // isz
    rin = torch.empty(nmax, dtype=tdt, device="cuda")
    rout = torch.empty_like(rin)
    stream = torch.cuda.current_stream()
    if a.nccl:
        cells = []
        for mib in a.mib:
            n = int(mib * (1 << 20)) // isz
            buf = rin[:n].clone()
            ms = bench.device_time_ms(lambda: dist.all_reduce(buf), a.iters, 5, stream, dist.barrier)
            t = torch.tensor([ms], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            cells.append(f"{mib:g}M:{bench.busbw(n * isz, world, t.item()):.0f}")
        if rank == 0:
            print(f"{'NCCL ' + os.environ.get('NCCL_ALGO', ''):40s} " + " ".join(cells), flush=True)
    for cfg in a.cfg:
        env = dict(kv.split("=", 1) for kv in cfg.split(",") if kv)
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        comm = lane.LaneComm(N, G, a.k, rank=rank, device=local)
        comm.register(rin)
        comm.register(rout)
        cells = []
        for mib in a.mib:
            n = int(mib * (1 << 20)) // isz
            inp = sdev.fill(rin[:n], a.dtype, "signed", 42, rank)
            out = rout[:n]
            ms = bench.device_time_ms(lambda: comm.allreduce(out, inp), a.iters, 5, stream, dist.barrier)
            ok = bench.sample_check([out], N, G, a.dtype, n, 42, [rank])
            t = torch.tensor([ms, 0.0 if ok else 1.0], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            pl = comm.plan(n, a.dtype)
            cells.append(f"{mib:g}M:{bench.busbw(n * isz, world, t[0].item()):.0f}"
                         f"{comm.protocol(n, a.dtype)[0]}{pl['ctas_per_group']}/{pl['chunk_granules']}"
                         f"{'' if t[1].item() == 0 else '!'}")
        if rank == 0:
            print(f"{cfg or 'default':40s} " + " ".join(cells), flush=True)
        torch.cuda.synchronize()
        dist.barrier()
        comm.close()
        dist.barrier()
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
