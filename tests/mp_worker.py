"""Multi-GPU parity worker: one process per GPU, launched by torchrun.

    torchrun --nproc-per-node P --master-addr 127.0.0.1 tests/mp_worker.py [--quick]

For every virtual layout N x G with N*G == P and several k, dtypes and
counts, rank p fills its sendbuf with the seeded generator, runs the lane
allreduce through LaneComm (C ABI, IPC peers over NVLink) and compares its
output element by element with the CPU oracle (bit-exact). The IPC handle
exchange uses a gloo process group. Exits non-zero on any mismatch.
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import oracle  # noqa: E402
import seeded_inputs as si  # noqa: E402
from seeded_inputs import device as sdev  # noqa: E402
import paper_2508_13397_b200 as lane  # noqa: E402
from tests.gpu_util import bits, to_numpy  # noqa: E402


def layouts(P):
    return [(N, P // N) for N in range(1, P + 1) if P % N == 0]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    os.environ.setdefault("LANE_TIMEOUT_MS", "10000")
    os.environ.setdefault("LANE_ROUND_BYTES", str(64 << 20))
    P = world
    counts = [1, 7, 4099, (1 << 20) + 3] if args.quick else [1, 7, 64, 4099, (1 << 20) + 3, (1 << 24) + 1]
    ks = [1, 4] if args.quick else [1, 2, 4, 8, 16]
    failures = 0
    t0 = time.time()
    maxb = max(counts) * 4
    cases = [(N, G, k, pr) for (N, G) in layouts(P) for k in ks
             for pr in ("simple", "dyn", "pull", "pullpush", "ll", "ll128", "ring2", "ring2_128")]
    if args.quick:  # the standard multi-PPG approach at PPG 16 (Alg. 1 per slice, P L431), both protocols
        cases += [(1, P, 16, "ll"), (1, P, 16, "ll128")]
    for N, G, k, proto in cases:
        if True:
            # ll / ll128: every call that fits that protocol's inboxes
            os.environ["LANE_PROTO"] = {"simple": "simple", "dyn": "simple", "pull": "simple", "pullpush": "simple",
                                        "ll128": "ll128", "ring2_128": "ll128"}.get(proto, "ll")
            if proto == "dyn":  # chunks claimed dynamically (forced; the default is by chunks per CTA)
                os.environ["LANE_DYN_CHUNKS"] = "1"
            else:
                os.environ.pop("LANE_DYN_CHUNKS", None)
            # registered job set: push / pull-all / pull-push
            os.environ["LANE_DIRECT"] = {"pull": "3", "pullpush": "4"}.get(proto, "2")
            if proto.startswith("ring2"):  # the lane method with Alg. 1 as its inter-node stage
                os.environ["LANE_PHASE2"] = "ring"
            else:
                os.environ.pop("LANE_PHASE2", None)
            comm = lane.LaneComm(N, G, k, rank=rank, device=local)
            # registered (zero-copy) buffers: one pair per comm, views at offset 0
            rin = torch.empty(maxb, dtype=torch.uint8, device="cuda")
            rout = torch.empty(maxb, dtype=torch.uint8, device="cuda")
            comm.register(rin)
            comm.register(rout)
            for dtype in ("int32", "float32", "bfloat16"):
                tdt = {"int32": torch.int32, "float32": torch.float32, "bfloat16": torch.bfloat16}[dtype]
                isz = torch.empty(0, dtype=tdt).element_size()
                for it, n in enumerate(counts * 2):
                    registered = it >= len(counts)
                    seed = 1000 + 17 * n + k + (7 if registered else 0)
                    if registered:
                        inp = sdev.fill(rin[:n * isz].view(tdt), dtype, "signed", seed, rank)
                    else:
                        inp = sdev.fill(torch.empty(n, dtype=tdt, device="cuda"), dtype, "signed", seed, rank)
                    inplace = it % 2 == 1
                    if inplace:
                        out = inp
                    else:
                        out = rout[:n * isz].view(tdt) if registered else torch.empty_like(inp)
                    comm.allreduce(out, inp)
                    torch.cuda.synchronize()
                    comm.check()
                    if n <= (1 << 20) + 3:
                        idx = np.arange(n)
                    else:
                        idx = si.sample_indices(n, 4099, [n // 2, n // 3])
                    xs = [si.generate_at(dtype, "signed", seed, p, idx) for p in range(P)]
                    if proto.startswith("ring2"):
                        if n > (1 << 20) + 3:  # sampled indices: the ring order needs whole chunks; exact int only
                            if dtype != "int32":
                                continue
                            ref = oracle.brute_force_sum(xs, dtype)
                        else:
                            pl = comm.plan(n, dtype)
                            assert pl["chunk_granules"] == 4096 and pl["round_granules"] == (16 << 20) // 16, pl
                            ref = oracle.lane_allreduce(xs, N, G, k, dtype, pl["chunk_granules"],
                                                        pl["round_granules"], phase2="ring").out[0]
                    else:
                        ref = oracle.lane_allreduce(xs, N, G, 1, dtype).out[0]
                    got = to_numpy(out[torch.from_numpy(idx).cuda()], dtype)
                    if not np.array_equal(bits(got), bits(ref)):
                        bad = np.nonzero(bits(got) != bits(ref))[0]
                        print(f"rank {rank} FAIL {proto} {N}x{G} k={k} {dtype} n={n} inplace={inplace} "
                              f"reg={registered}: "
                              f"{len(bad)} mismatches first {idx[bad[:5]]}", flush=True)
                        failures += 1
            # ring allreduce (Alg. 1) vs the ring oracle, on the same comm (LL packets / LL128 lines)
            if proto in ("ll", "ll128"):
                for dtype, n in (("float32", 4099), ("bfloat16", (1 << 20) + 3), ("int32", 7)):
                    tdt = {"int32": torch.int32, "float32": torch.float32, "bfloat16": torch.bfloat16}[dtype]
                    inp = sdev.fill(torch.empty(n, dtype=tdt, device="cuda"), dtype, "signed", 5 + n, rank)
                    out = torch.empty_like(inp)
                    comm.allreduce_ring(out, inp)
                    torch.cuda.synchronize()
                    comm.check()
                    xs = [si.generate(dtype, "signed", 5 + n, p_, n) for p_ in range(P)]
                    pl = comm.plan(n, dtype, algorithm="ring")
                    # R#21: the ring geometry is fixed by the env, never by the launch
                    assert pl["chunk_granules"] == 4096 and pl["round_granules"] == (16 << 20) // 16, pl
                    ref = oracle.ring_allreduce(xs, k, dtype, pl["chunk_granules"], pl["round_granules"]).out[0]
                    if not np.array_equal(bits(to_numpy(out, dtype)), bits(ref)):
                        print(f"rank {rank} FAIL ring {N}x{G} k={k} {dtype} n={n}", flush=True)
                        failures += 1
            # "approach 2" (P L296-297) vs its oracle (= the lane method's bits)
            if proto == "ll":
                for dtype, n in (("float32", 4099), ("bfloat16", (1 << 20) + 3)):
                    tdt = {"float32": torch.float32, "bfloat16": torch.bfloat16}[dtype]
                    inp = sdev.fill(torch.empty(n, dtype=tdt, device="cuda"), dtype, "signed", 9 + n, rank)
                    out = torch.empty_like(inp)
                    comm.allreduce_approach2(out, inp)
                    torch.cuda.synchronize()
                    comm.check()
                    xs = [si.generate(dtype, "signed", 9 + n, p_, n) for p_ in range(P)]
                    ref = oracle.approach2_allreduce(xs, N, G, k, dtype).out[0]
                    if not np.array_equal(bits(to_numpy(out, dtype)), bits(ref)):
                        print(f"rank {rank} FAIL approach2 {N}x{G} k={k} {dtype} n={n}", flush=True)
                        failures += 1
            # host-buffer API (pipelined pieces, ragged tail; each piece is its own
            # allreduce, so only the direct stage's order is piece-independent)
            if proto.startswith("ring2"):
                dist.barrier()
                comm.close()
                dist.barrier()
                continue
            os.environ["LANE_HOST_PIECE_BYTES"] = str(1 << 18)
            n = (1 << 20) + 5
            hx = si.generate("float32", "signed", 77 + k, rank, n)
            hin = torch.from_numpy(hx).pin_memory()
            hout = torch.empty_like(hin).pin_memory()
            comm.allreduce_host(hout, hin)
            ref = oracle.lane_allreduce([si.generate("float32", "signed", 77 + k, p_, n) for p_ in range(P)],
                                        N, G, 1, "float32").out[0]
            if not np.array_equal(hout.numpy().view(np.uint32), ref.view(np.uint32)):
                print(f"rank {rank} FAIL host api {N}x{G} k={k}", flush=True)
                failures += 1
            os.environ.pop("LANE_HOST_PIECE_BYTES")
            dist.barrier()
            comm.close()
            dist.barrier()
    failures += graph_cases(P, rank, local)
    ok = torch.tensor([failures])
    dist.all_reduce(ok)
    if rank == 0:
        print(f"mp_worker P={P}: {'OK' if ok.item() == 0 else 'FAILED'} ({ok.item()} failures) "
              f"in {time.time() - t0:.1f}s", flush=True)
    dist.destroy_process_group()
    sys.exit(1 if ok.item() else 0)


def graph_cases(P, rank, local):
    """CUDA graphs: every rank captures the same three calls (simple on
    registered buffers, LL, LL128) into a graph and replays it three times
    with fresh inputs (device-side epochs, lane_kernels.cuh launch_prologue),
    with an eager call between replays; bit-exact vs the oracle."""
    failures = 0
    for (N, G) in layouts(P):
        os.environ.pop("LANE_PROTO", None)
        os.environ.pop("LANE_PHASE2", None)
        os.environ.pop("LANE_DYN_CHUNKS", None)
        os.environ["LANE_LL128_THRESHOLD_BYTES"] = str(2 << 20)  # 4 MiB: simple protocol
        os.environ["LANE_LL_THRESHOLD_BYTES"] = str(64 << 10)
        os.environ["LANE_LL128_MIN_BYTES"] = str(512 << 10)  # 1 MiB: LL128 at every P
        comm = lane.LaneComm(N, G, 1, rank=rank, device=local)
        sizes = [(1 << 20) + 5, 3000, (1 << 18) + 3]
        rin = torch.empty(4 * sizes[0], dtype=torch.uint8, device="cuda")
        rout = torch.empty_like(rin)
        comm.register(rin)
        comm.register(rout)
        ins = [rin[:4 * sizes[0]].view(torch.float32)] + [torch.empty(n, device="cuda") for n in sizes[1:]]
        outs = [rout[:4 * sizes[0]].view(torch.float32)] + [torch.empty(n, device="cuda") for n in sizes[1:]]
        protos = [comm.protocol(n, "float32") for n in sizes]
        assert protos == ["simple", "ll", "ll128"], protos
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            g.capture_begin()
            for i_, o_ in zip(ins, outs):
                comm.allreduce(o_, i_)
            g.capture_end()
        torch.cuda.current_stream().wait_stream(s)
        for rep in range(3):
            seed = 3100 + rep
            for t, n in zip(ins, sizes):
                sdev.fill(t, "float32", "signed", seed + n, rank)
            torch.cuda.synchronize()
            dist.barrier()
            g.replay()
            torch.cuda.synchronize()
            comm.check()
            for o, n, pr in zip(outs, sizes, protos):
                xs = [si.generate("float32", "signed", seed + n, p_, n) for p_ in range(P)]
                ref = oracle.lane_allreduce(xs, N, G, 1, "float32").out[0]
                if not np.array_equal(bits(to_numpy(o, "float32")), bits(ref)):
                    print(f"rank {rank} FAIL graph {N}x{G} replay {rep} n={n} proto={pr}", flush=True)
                    failures += 1
            n = 4099 + rep  # an eager call between replays
            inp = sdev.fill(torch.empty(n, device="cuda"), "float32", "signed", 77 + rep, rank)
            out = torch.empty_like(inp)
            comm.allreduce(out, inp)
            torch.cuda.synchronize()
            comm.check()
            xs = [si.generate("float32", "signed", 77 + rep, p_, n) for p_ in range(P)]
            ref = oracle.lane_allreduce(xs, N, G, 1, "float32").out[0]
            if not np.array_equal(bits(to_numpy(out, "float32")), bits(ref)):
                print(f"rank {rank} FAIL graph-mode eager {N}x{G} rep {rep}", flush=True)
                failures += 1
        os.environ.pop("LANE_LL128_THRESHOLD_BYTES")
        os.environ.pop("LANE_LL_THRESHOLD_BYTES")
        os.environ.pop("LANE_LL128_MIN_BYTES")
        dist.barrier()
        del g
        comm.close()
        dist.barrier()
    return failures


if __name__ == "__main__":
    main()
