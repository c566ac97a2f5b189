"""P ranks on ONE GPU (P processes, all on cuda:0) exercising the multi-GPU
code path — IPC-mapped peer memory (same-device IPC handles), system-scope
epoch flags, the start handshake with the call signature and the end barrier,
registered (zero-copy) and staged buffers — on a box with a single GPU, where
the kernels of the P processes share the GPU (every cross-rank wait is
bounded by the watchdog). LANE_TEST_GPUS=g spreads the ranks over g GPUs
(rank % g), so P = 8 runs on a 1- or 2-GPU box, some peers local and some over
NVLink. Every layout N x G of P, k = 1 and 2, simple /
bulk stores / chunk claims / LL / LL128, fp32 / bf16 / int32, 5 to 2^20 + 3
elements.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tests/mp_samedev_worker.py

Prints ``mp_samedev_worker: OK`` when every output element matches the oracle.
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import oracle  # noqa: E402
import seeded_inputs as si  # noqa: E402
from seeded_inputs import device as sdev  # noqa: E402
import paper_2508_13397_b200 as lane  # noqa: E402
from tests.gpu_util import bits, to_numpy  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = rank % int(os.environ.get("LANE_TEST_GPUS", "1"))  # > 1: some peers local, some over NVLink
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")
    os.environ.setdefault("LANE_TIMEOUT_MS", "60000")
    t0 = time.time()
    failures = 0
    layouts = [(N, world // N) for N in range(1, world + 1) if world % N == 0]
    protos = ("simple", "simple-bulk", "simple-claims", "ll", "ll128")
    ks = (1, 2)
    if "--quick" in sys.argv:  # P = 8 on one or two GPUs: every layout and protocol, fewer k
        ks = (1,)
    cases = [(N, G, k, proto) for (N, G) in layouts for k in ks for proto in protos]
    tdts = {"int32": torch.int32, "float32": torch.float32, "bfloat16": torch.bfloat16}
    for N, G, k, proto in cases:
        os.environ["LANE_PROTO"] = proto.split("-")[0]
        os.environ["LANE_STORE"] = "bulk" if proto == "simple-bulk" else "auto"
        os.environ["LANE_DYN_CHUNKS"] = "1" if proto == "simple-claims" else "-1"
        comm = lane.LaneComm(N, G, k, rank=rank, device=dev)
        n_max = (1 << 20) + 3
        rin = torch.empty(4 * n_max, dtype=torch.uint8, device="cuda")
        rout = torch.empty_like(rin)
        comm.register(rin)
        comm.register(rout)
        for dtype in ("float32", "bfloat16", "int32"):
            tdt = tdts[dtype]
            for n in (5, 4099, n_max):
                for registered in (False, True):
                    seed = 4000 + n + (7 if registered else 0) + k
                    isz = tdt.itemsize
                    inp = rin[:n * isz].view(tdt) if registered else torch.empty(n, dtype=tdt, device="cuda")
                    sdev.fill(inp, dtype, "signed", seed, rank)
                    out = rout[:n * isz].view(tdt) if registered else torch.empty_like(inp)
                    comm.allreduce(out, inp)
                    torch.cuda.synchronize()
                    comm.check()
                    xs = [si.generate(dtype, "signed", seed, p, n) for p in range(world)]
                    ref = oracle.lane_allreduce(xs, N, G, k, dtype).out[0]
                    if not np.array_equal(bits(to_numpy(out, dtype)), bits(ref)):
                        print(f"rank {rank} FAIL {N}x{G} k={k} {proto} {dtype} n={n} registered={registered}",
                              flush=True)
                        failures += 1
        dist.barrier()
        comm.close()
        dist.barrier()
    ok = torch.tensor([failures])
    dist.all_reduce(ok)
    if rank == 0:
        print(f"mp_samedev_worker: {'OK' if ok.item() == 0 else 'FAILED'} ({ok.item()} failures) "
              f"in {time.time() - t0:.1f}s", flush=True)
    dist.destroy_process_group()
    sys.exit(1 if ok.item() else 0)


if __name__ == "__main__":
    main()
