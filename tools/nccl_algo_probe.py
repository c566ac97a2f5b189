"""Which algorithm NCCL picks for a 1 GiB fp32 allreduce on this box when
NCCL_ALGO is unset (the bench's "nccl_default_context" comparator), and
whether NVLS (NVLink SHARP) is available: one torchrun job with NCCL's own
INIT / NVLS / TUNING log, then the measured busbw of the default and of
NCCL_ALGO=Ring / NVLS / Tree communicators created one after the other (NCCL
reads NCCL_ALGO when a communicator is created). Dev tool; writes the log to
$NCCL_DEBUG_FILE if set.

    NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,NVLS,TUNING torchrun --nproc-per-node 4 tools/nccl_algo_probe.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    os.environ.pop("NCCL_ALGO", None)
    dist.init_process_group("cpu:gloo,cuda:nccl")
    import bench  # noqa: E402  (after init: bench sets NCCL_ALGO=Ring as a default for its own runs)
    os.environ.pop("NCCL_ALGO", None)
    n = (1 << 30) // 4
    buf = torch.ones(n, device="cuda")
    stream = torch.cuda.current_stream()
    rows = []
    for algo in (None, "Ring", "NVLS", "Tree"):
        if algo:
            os.environ["NCCL_ALGO"] = algo
        else:
            os.environ.pop("NCCL_ALGO", None)
        try:
            g = dist.new_group(backend="nccl")
            dist.all_reduce(buf[:1024], group=g)
            torch.cuda.synchronize()
            ms = bench.max_over_ranks(bench.device_time_ms(lambda: dist.all_reduce(buf, group=g), 10, 3, stream,
                                                           lambda: dist.barrier()))
            rows.append({"algo": algo or "default", "ms": round(ms, 4), "busbw": round(bench.busbw(n * 4, world, ms), 2)})
        except Exception as e:  # an algorithm NCCL cannot run here
            rows.append({"algo": algo, "error": str(e)[:200]})
    if rank == 0:
        for r in rows:
            print(json.dumps(dict(r, P=world, bytes=n * 4)), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
