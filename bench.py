"""Benchmark of the k-split multi-lane allreduce (arXiv 2508.13397) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W]                 # our arm
    python bench.py --impl reference ...                                 # CPU oracle arm
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

Metric (BASELINE.json): allreduce bus GB/s (busbw = S/t * 2(P-1)/P, t =
device time per call, max over ranks) vs message size at 2/4/8 B200, vs NCCL
ring, and % of the NVLink roofline.

N = 1: the headline layout (2 virtual nodes x 4 GPUs, k = 1, fp32, 1 GiB per
rank; BASELINE configs[1] at its largest size) EMULATED on one B200: all 8
ranks' buffers live in this GPU's HBM and one cooperative launch of the same
kernel runs every rank (lane_allreduce_emulated). The bound is then HBM.
N > 1: one process per GPU (torchrun), real IPC/NVLink; default layout
2 x (N/2) virtual nodes, k = 1, fp32, 1 GiB per rank. Bound: NVLink.

One JSON line is printed by rank 0. Each timed step is one lane_allreduce call
(one kernel launch per round; one round at these sizes) on inputs already in
HBM; inputs are 1 GiB per rank (> 126 MB L2), so no L2 flush is needed.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# NCCL is used ONLY for the timed comparator; the required comparator is ring.
os.environ.setdefault("NCCL_ALGO", "Ring")
# NCCL's version banner goes to stdout; the contract is ONE JSON line from rank 0
if os.environ.get("NCCL_DEBUG", "").upper() in ("VERSION", "WARN"):
    os.environ.pop("NCCL_DEBUG")

METRIC = "allreduce bus GB/s vs msg size at 2/4/8 B200 vs NCCL ring; % of NVLink roofline"
NVLINK_PEAK = 770.0  # GB/s per direction per GPU, measured peer copy (B200_PROFILING.md)
NVLINK_NOMINAL = 900.0
TDT = {"int32": "int32", "float32": "float32", "bfloat16": "bfloat16"}
SHORT = {"int32": "i32", "float32": "f32", "bfloat16": "bf16"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="lane", choices=["lane", "reference"])
    ap.add_argument("--layout", default=None, help="NxG virtual layout (default 2x4 / 2x(N/2))")
    ap.add_argument("--k", type=int, default=1, help="procs per GPU = CTA groups")
    ap.add_argument("--dtype", default="float32", choices=list(TDT))
    ap.add_argument("--mib", type=float, default=1024.0, help="message MiB per rank")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-nccl", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--nccl-ppg", type=int, default=4,
                    help="multi-GPU: also time the paper's multi-PPG CCL variant (P L269, L504): this many "
                         "NCCL communicators, each allreducing a 1/PPG slice on its own stream (0 = skip)")
    ap.add_argument("--no-register", action="store_true",
                    help="multi-GPU: do not register the buffers (staged path through library scratch)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--ring", action="store_true",
                    help="sweep: also time the library's ring allreduce (Alg. 1, the paper's standard algorithm)")
    ap.add_argument("--approach2", action="store_true",
                    help="sweep: also time the paper's draft 'approach 2' (node allreduce + lane allreduce)")
    ap.add_argument("--sweep", default=None,
                    help="multi-GPU: write busbw vs message size (ours and NCCL ring) as JSONL to this file")
    return ap.parse_args()


# ----------------------------------------------------------------- helpers
def itemsize(dtype):
    return 2 if dtype == "bfloat16" else 4


def max_over_ranks(ms):
    """Device time of a multi-rank step: the MAX over ranks (every rank gets
    it; torch.distributed, gloo or nccl)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(ms)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def busbw(bytes_, P, ms):
    return bytes_ * 2 * (P - 1) / P / (ms * 1e-3) / 1e9 if P > 1 else bytes_ / (ms * 1e-3) / 1e9


class Clocks:
    """nvidia-smi sampler running while the timed region runs."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpus):
        self.gpus = gpus
        self.proc = None
        self.out = os.path.join("/tmp", f"lane_clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            self.f = open(self.out, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", ",".join(str(g) for g in self.gpus)], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()
            self.f.close()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            for line in open(self.out):
                f = [x.strip() for x in line.split(",")]
                if len(f) < 8:
                    continue
                try:
                    sm.append(float(f[1]))
                    mx.append(float(f[2]))
                except ValueError:
                    continue
                for nm, v in zip(names, f[4:8]):
                    if v.lower().startswith("active"):
                        reasons.add(nm)
        except OSError:
            pass
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def device_time_ms(fn, steps, warmup, stream, barrier=None):
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    if barrier:
        barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream)
    for _ in range(steps):
        fn()
    e.record(stream)
    torch.cuda.synchronize()
    if barrier:
        barrier()
    return s.elapsed_time(e) / steps


def nvlink_bytes(dev):
    try:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        from nvlink_counters import nvlink_bytes as nb
        return nb(dev)
    except Exception:
        return None


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


def method_hbm_bytes(N, G, S):
    """Compulsory HBM bytes per rank of the three-phase method when every rank's
    buffers share one HBM (emulated mode; SURVEY §8(d) "HBM: >= 3.1 d, pull
    design"): read the inputs (S), materialise and re-read the phase-1 result T1
    (S/G each way), write the lane result into the lane members' recvbufs (S/G),
    and the phase-3 allgather re-reads and writes the node's other parts
    ((G-1)/G S each way): S (3 + 1/G). With G = 1 there is no phase 1 or 3 and
    the floor is the allreduce's own 2 S."""
    return 2 * S if G == 1 else int(S * (3 + 1 / G))


def ncu_traffic(layout, k, dtype, S, P):
    """DRAM bytes per launch from the committed ncu summary of this workload
    (profiles/*ncu*summary.json); scaled linearly from the captured size when
    the captured message size differs. None if there is no capture."""
    import glob
    best = None
    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", "*ncu*summary.json"))):
        try:
            d = json.load(open(f))
        except (OSError, ValueError):
            continue
        w = d.get("workload", "")
        names = {dtype, SHORT[dtype], "fp32" if dtype == "float32" else dtype}
        if not (w.startswith(layout + " ") and f"k={k}" in w and any(nm in w for nm in names)):
            continue
        kern = [x for x in d.get("kernels", []) if "lane_tma" in x.get("kernel", "")]
        if not kern or "dram_bytes_per_rank_per_byte" not in kern[0]:
            continue
        cand = (abs(d["bytes_per_rank"] - S), f, kern[0]["dram_bytes_per_rank_per_byte"], d["bytes_per_rank"])
        best = cand if best is None or cand < best else best
    if best is None:
        return None, None
    _, f, per, captured = best
    note = os.path.basename(f) + ("" if captured == S else f" (scaled from {captured >> 20} MiB/rank)")
    return int(per * S * P), note


def cpu_baseline(N, G, k, dtype, seconds):
    """The oracle as it stands, on this host, single-threaded numpy, on a
    bounded sample of the workload (same layout/dtype, 2^20 elements per rank)."""
    import oracle
    import seeded_inputs as si
    n = 1 << 20
    xs = si.generate_all(dtype, "signed", 42, N * G, n)
    t0 = time.perf_counter()
    reps = 0
    while True:
        oracle.lane_allreduce(xs, N, G, k, dtype)
        reps += 1
        el = time.perf_counter() - t0
        if el >= seconds or reps >= 200:
            break
    t = el / reps
    S = n * itemsize(dtype)
    return {"value": round(busbw(S, N * G, t * 1e3), 4), "unit": "GB/s", "cores": 1, "kind": "oracle",
            "host_cores": os.cpu_count(),
            "sample": f"{N}x{G} k={k} {dtype}, {n} elements ({S >> 20} MiB) per simulated rank, "
                      f"{reps} reps in {el:.1f}s, {t * 1e3:.1f} ms per oracle allreduce (numpy, 1 thread)"}


# ----------------------------------------------------------------- in-run verification
# bench.py checks its own outputs without the oracle (only the cpu_baseline leg
# and the reference arm run oracle/): the plain definition of the sum, and the
# canonical reduction order written out here for sampled positions.
TOLERANCE = {"float32": 1e-6, "bfloat16": 1e-2}  # north_star, relative to sum |x| (DESIGN R#10)


def _f32(a, dtype):
    """Stored values -> float32 (bf16 bits widened exactly)."""
    import numpy as np
    if dtype == "bfloat16":
        return (np.asarray(a, np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)
    return np.asarray(a, np.float32)


def _bf16_rne(f):
    """float32 -> bf16 bits, round to nearest even (finite values)."""
    import numpy as np
    u = np.asarray(f, np.float32).view(np.uint32).astype(np.uint64)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


def canonical_lane_sum(xs, N, G, dtype):
    """The lane method's result in its canonical order (DESIGN R#7, R#8): node
    sums over h = 0..G-1 in order (fp32 accumulate, bf16 rounded once), then
    the sum of the N node sums over a = 0..N-1 in order (rounded once); int32
    wraps mod 2^32. xs[p] = rank p's values at the sampled positions."""
    import numpy as np
    if dtype == "int32":
        s = np.zeros(len(xs[0]), np.int64)
        for x in xs:
            s += np.asarray(x, np.int64)
        return (s & 0xFFFFFFFF).astype(np.uint32).view(np.int32)
    node = []
    for a in range(N):
        acc = _f32(xs[a * G], dtype).copy()
        for h in range(1, G):
            acc = (acc + _f32(xs[a * G + h], dtype)).astype(np.float32)
        node.append(_f32(_bf16_rne(acc), dtype) if dtype == "bfloat16" else acc)
    acc = node[0].copy()
    for a in range(1, N):
        acc = (acc + node[a]).astype(np.float32)
    return _bf16_rne(acc) if dtype == "bfloat16" else acc


def _within_tolerance(got, xs, dtype, tol):
    """int32: exact plain sum mod 2^32; fp: |got - sum| <= tol * sum |x| (float64)."""
    import numpy as np
    if dtype == "int32":
        return np.array_equal(np.asarray(got, np.int32), canonical_lane_sum(xs, 1, len(xs), dtype))
    ref = np.zeros(len(xs[0]), np.float64)
    mag = np.zeros(len(xs[0]), np.float64)
    for x in xs:
        v = _f32(x, dtype).astype(np.float64)
        ref += v
        mag += np.abs(v)
    return bool(np.all(np.abs(_f32(got, dtype).astype(np.float64) - ref) <= tol * mag * (1 + 1e-9)))


def _host_values(t, dtype):
    import torch
    t = t.cpu()
    return t.view(torch.int16).numpy().view("uint16") if dtype == "bfloat16" else t.numpy()


def sample_check(outs, N, G, dtype, n, seed, ranks):
    """Sampled outputs bit-exact against the canonical order (canonical_lane_sum).
    With LANE_PHASE2=ring (DESIGN R#22) an element's ring order depends on its
    whole chunk, which a sample does not carry: there int32 is checked exactly
    and fp within the north_star tolerance; the bit-exact ring-variant parity
    is in tests/."""
    import numpy as np
    import torch
    import seeded_inputs as si
    idx = si.sample_indices(n, 65537, [n // 2, n // 3, n // 5])
    it = torch.from_numpy(idx).to(outs[0].device)
    xs = [si.generate_at(dtype, "signed", seed, p, idx) for p in range(N * G)]
    if os.environ.get("LANE_PHASE2") == "ring" and N > 2:
        return all(_within_tolerance(_host_values(o[it], dtype), xs, dtype, TOLERANCE.get(dtype, 0.0)) for o in outs)
    ref = canonical_lane_sum(xs, N, G, dtype)
    vb = np.uint16 if dtype == "bfloat16" else np.uint32
    return all(np.array_equal(_host_values(o[it], dtype).view(vb), ref.view(vb)) for o in outs)


def ring_check(out, P, k, dtype, n, seed, plan):
    """Check of the ring allreduce's output (Alg. 1 order, per-hop rounding) on
    the first 2^16 elements: int32 exact, fp within the per-hop error bound
    (P-1 roundings, plus one bf16 rounding per hop). Bit-exact ring parity
    against the ring oracle is in tests/."""
    import numpy as np
    import seeded_inputs as si
    m = min(n, 1 << 16)
    idx = np.arange(m)
    xs = [si.generate_at(dtype, "signed", seed, p, idx) for p in range(P)]
    u = 2.0 ** -24 + (2.0 ** -8 if dtype == "bfloat16" else 0.0)
    return _within_tolerance(_host_values(out[:m], dtype), xs, dtype, (P - 1) * u)


def base_line(args, N_gpus, K, W):
    return {"metric": METRIC, "unit": "GB/s", "n_gpus": N_gpus, "steps": K, "warmup": W,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": SHORT[args.dtype]}


# ----------------------------------------------------------------- reference arm
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    import seeded_inputs as si
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    N, G = layout_for(args, max(world, args.gpus))
    n = 1 << 18  # bounded sample per rank per step
    xs = si.generate_all(args.dtype, "signed", 42, N * G, n)
    for _ in range(args.warmup):
        oracle.lane_allreduce(xs, N, G, args.k, args.dtype)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.lane_allreduce(xs, N, G, args.k, args.dtype)
    t = (time.perf_counter() - t0) / args.steps
    S = n * itemsize(args.dtype)
    v = round(busbw(S, N * G, t * 1e3), 4)
    line = base_line(args, args.gpus, args.steps, args.warmup)
    line.update({"impl": "reference", "value": v, "ms_per_step": round(t * 1e3, 3),
                 "data": "synthetic (seeded counter hash)",
                 "config": {"workload": f"CPU oracle, {N}x{G} virtual ranks, k={args.k}, {args.dtype}, "
                                        f"{S >> 10} KiB per rank per step (bounded sample of the "
                                        f"{int(args.mib)} MiB workload)",
                            "layout": f"{N}x{G}", "procs_per_gpu": args.k},
                 "cpu_baseline": {"value": v, "unit": "GB/s", "cores": 1, "kind": "oracle",
                                  "host_cores": os.cpu_count(),
                                  "sample": f"{n} elements per simulated rank per step"},
                 "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                 "gpu_launches": 0})
    print(json.dumps(line), flush=True)
    return 0


def layout_for(args, P):
    if args.layout:
        N, G = map(int, args.layout.lower().split("x"))
        return N, G
    if P == 1:
        return 2, 4  # emulated headline layout
    if P % 2 == 0:
        return 2, P // 2
    return P, 1


# ----------------------------------------------------------------- N = 1 (emulated)
def run_single(args):
    import torch
    import paper_2508_13397_b200 as lane
    from seeded_inputs import device as sdev
    N, G = layout_for(args, 1)
    P, k, dtype = N * G, args.k, args.dtype
    isz = itemsize(dtype)
    n = int(args.mib * (1 << 20)) // isz
    S = n * isz
    torch.cuda.set_device(0)
    tdt = getattr(torch, dtype)
    emu = lane.LaneEmulator(N, G, k, device=0)
    plan = emu.plan(n, dtype)
    seed = 42
    ins = [sdev.fill(torch.empty(n, dtype=tdt, device="cuda:0"), dtype, "signed", seed, p) for p in range(P)]
    outs = [torch.empty_like(t) for t in ins]
    stream = torch.cuda.current_stream()
    step = lambda: emu.allreduce(outs, ins)  # noqa: E731
    with Clocks([0]) as clk:
        ms = device_time_ms(step, args.steps, args.warmup, stream)
    emu.check()
    ok = sample_check(outs, N, G, dtype, n, seed, range(P))
    # roofline: HBM. Algorithmic bytes per launch = the method's compulsory
    # HBM traffic with all P ranks in one HBM (method_hbm_bytes);
    # the plain allreduce floor 2*P*S is reported beside it.
    pk = peaks()
    hbm_peak = float(pk.get("hbm_gbs", 6650.0))
    launches = max(plan["launches"], 1)
    algo = P * method_hbm_bytes(N, G, S)
    achieved = algo / launches / (ms / launches * 1e-3) / 1e9
    traffic, traffic_src = ncu_traffic(f"{N}x{G}", k, dtype, S, P)
    line = base_line(args, 1, args.steps, args.warmup)
    bw = busbw(S, P, ms)
    line.update({
        "value": round(bw, 2) if ok else None, "ms_per_step": round(ms, 4),
        "data": "synthetic (seeded counter hash; signed values)",
        "config": {"workload": f"{N}x{G} virtual ranks emulated on 1 B200 (all ranks in one cooperative "
                               f"launch), k={k}, {dtype}, {S >> 20} MiB per rank (BASELINE configs[1] layout "
                               f"at its largest size)",
                   "layout": f"{N}x{G}", "procs_per_gpu": k, "bytes_per_rank": S, "emulated": True,
                   "protocol": emu.protocol(n, dtype),
                   "l2": (f"inputs larger than L2 ({P} x {S >> 20} MiB)" if P * S > (126 << 20)
                          else "inputs fit in L2; not flushed"), "plan": plan},
        "algbw": round(S / (ms * 1e-3) / 1e9, 2),
        "verified": ok,
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                     "frac": round(achieved / hbm_peak, 4),
                     "traffic": None if traffic is None else traffic // launches,
                     "traffic_source": traffic_src,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy)" if "hbm_gbs" in pk
                     else "fallback guide",
                     "algorithmic_bytes_per_launch": algo // launches,
                     "algorithmic_basis": "method compulsory HBM bytes, P ranks in one HBM: S(3+1/G) per rank",
                     "allreduce_floor_bytes_per_launch": 2 * P * S // launches,
                     "frac_of_allreduce_floor": round(2 * P * S / (ms * 1e-3) / 1e9 / hbm_peak, 4)},
        "gpu_launches": args.steps * launches,
        "clocks": clk.summary(),
    })
    if not args.no_e2e:
        line["e2e"] = e2e_single(emu, ins, outs, N, G, dtype, n, S, args)
    if not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(N, G, k, dtype, args.cpu_seconds)
    print(json.dumps(line), flush=True)
    return 0 if ok else 1


def e2e_single(emu, ins, outs, N, G, dtype, n, S, args):
    import torch
    P = N * G
    h_in = [torch.empty(n, dtype=ins[0].dtype).pin_memory() for _ in range(P)]
    h_out = [torch.empty(n, dtype=ins[0].dtype).pin_memory() for _ in range(P)]
    for h, d in zip(h_in, ins):
        h.copy_(d)
    stream = torch.cuda.current_stream()
    step = lambda: emu.allreduce_host(h_out, h_in)  # noqa: E731  (H2D + kernel + D2H, then sync)
    ms = device_time_ms(step, args.e2e_steps, 1, stream)
    return {"value": round(busbw(S, P, ms), 2), "unit": "GB/s", "ms_per_step": round(ms, 3),
            "h2d_bytes_per_step": P * S, "d2h_bytes_per_step": P * S,
            "api": "lane_allreduce_emulated_host (C ABI, pinned host buffers)"}


# ----------------------------------------------------------------- N > 1
def run_multi(args):
    import torch
    import torch.distributed as dist
    import paper_2508_13397_b200 as lane
    from seeded_inputs import device as sdev
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("cpu:gloo,cuda:nccl")
    N, G = layout_for(args, world)
    if N * G != world:
        raise SystemExit(f"layout {N}x{G} does not match world size {world}")
    P, k, dtype = world, args.k, args.dtype
    isz = itemsize(dtype)
    n = int(args.mib * (1 << 20)) // isz
    S = n * isz
    tdt = getattr(torch, dtype)
    comm = lane.LaneComm(N, G, k, rank=rank, device=local)
    plan = comm.plan(n, dtype)
    seed = 42
    inp = sdev.fill(torch.empty(n, dtype=tdt, device="cuda"), dtype, "signed", seed, rank)
    out = torch.empty_like(inp)
    registered = not args.no_register
    if registered:  # zero-copy: the paper shares the user buffer via IPC handles (P L330)
        comm.register(inp)
        comm.register(out)
    stream = torch.cuda.current_stream()
    barrier = lambda: dist.barrier()  # noqa: E731
    step = lambda: comm.allreduce(out, inp)  # noqa: E731
    clk = Clocks(list(range(world))) if rank == 0 else None
    if clk:
        clk.__enter__()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    nv0 = nvlink_bytes(local)
    ms = device_time_ms(step, args.steps, 0, stream, barrier)
    nv1 = nvlink_bytes(local)
    if clk:
        clk.__exit__()
    comm.check()
    ms_max = max_over_ranks(ms)
    ok = sample_check([out], N, G, dtype, n, seed, [rank])
    okt = torch.tensor([0 if ok else 1])
    dist.all_reduce(okt)
    ok = okt.item() == 0
    bw = busbw(S, P, ms_max)
    launches = max(plan["launches"], 1)
    # measured NVLink data bytes per launch (NVML counters of this GPU), mean over ranks
    nv = torch.tensor([-1.0, -1.0], dtype=torch.float64)
    if nv0 and nv1:
        nv = torch.tensor([(nv1[0] - nv0[0]) / (args.steps * launches), (nv1[1] - nv0[1]) / (args.steps * launches)],
                          dtype=torch.float64)
    nvs = [torch.zeros(2, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(nvs, nv)
    tx = [float(v[0]) for v in nvs]
    rx = [float(v[1]) for v in nvs]
    nvl = None if min(tx) < 0 else {"tx_bytes_per_launch_mean": sum(tx) / world,
                                     "rx_bytes_per_launch_mean": sum(rx) / world,
                                     "tx_over_algorithmic": sum(tx) / world / (2 * (P - 1) / P * S / launches)}
    line = base_line(args, world, args.steps, args.warmup)
    line.update({
        "value": round(bw, 2) if ok else None, "ms_per_step": round(ms_max, 4),
        "data": "synthetic (seeded counter hash; signed values)",
        "config": {"workload": f"{N}x{G} virtual nodes on {world} B200 (one process per GPU, IPC peers over "
                               f"NVLink 5), k={k}, {dtype}, {S >> 20} MiB per rank",
                   "layout": f"{N}x{G}", "procs_per_gpu": k, "bytes_per_rank": S, "emulated": False,
                   "registered_buffers": registered, "protocol": comm.protocol(n, dtype),
                   "l2": (f"inputs larger than L2 ({S >> 20} MiB per rank)" if S > (126 << 20)
                          else f"inputs ({S >> 20} MiB per rank) fit in L2; not flushed"), "plan": plan},
        "algbw": round(S / (ms_max * 1e-3) / 1e9, 2),
        "verified": ok,
        "roofline": {"bound": "nvlink", "achieved": round(bw, 2), "peak": NVLINK_PEAK, "unit": "GB/s",
                     "frac": round(bw / NVLINK_PEAK, 4), "frac_of_nominal_900": round(bw / NVLINK_NOMINAL, 4),
                     "traffic": None if nvl is None else int(nvl["tx_bytes_per_launch_mean"]),
                     "traffic_source": "NVML NVLink data TX counters (mean over ranks; ncu cannot wrap "
                                       "multi-rank runs)" if nvl else None,
                     "nvlink_counters": nvl,
                     "peak_source": "measured peer copy per direction, B200_PROFILING.md (no NVLink entry in "
                                    "MEASURED_PEAKS.json)",
                     "algorithmic_bytes_per_launch": int(2 * (P - 1) / P * S / launches)},
        "gpu_launches": args.steps * launches,
    })
    if clk:
        line["clocks"] = clk.summary()
    if not args.no_e2e:
        line["e2e"] = e2e_multi(comm, inp, N, G, dtype, n, S, args, dist)
    if not args.no_nccl:
        line["nccl_ring"] = nccl_ring(inp, S, P, args, dist, stream)
        if args.nccl_ppg > 1:
            line["nccl_ring_multi_ppg"] = nccl_ppg(inp, S, P, args, dist, stream, NcclPPG(args.nccl_ppg, dist))
    if rank == 0:
        print(json.dumps(line), flush=True)
    comm.close()
    dist.barrier()
    dist.destroy_process_group()
    return 0 if ok else 1


def e2e_multi(comm, inp, N, G, dtype, n, S, args, dist):
    import torch
    h_in = torch.empty(n, dtype=inp.dtype).pin_memory()
    h_in.copy_(inp)
    h_out = torch.empty_like(h_in).pin_memory()
    stream = torch.cuda.current_stream()
    ms = device_time_ms(lambda: comm.allreduce_host(h_out, h_in), args.e2e_steps, 1, stream,
                        lambda: dist.barrier())
    ms = max_over_ranks(ms)
    P = N * G
    return {"value": round(busbw(S, P, ms), 2), "unit": "GB/s", "ms_per_step": round(ms, 3),
            "h2d_bytes_per_step": S, "d2h_bytes_per_step": S,
            "api": "lane_allreduce_host (C ABI, pinned host buffers)"}


class NcclPPG:
    """the paper's multi-PPG CCL approach — PPG communicators per
    GPU, each running a standard NCCL allreduce on its own 1/PPG slice of the
    buffer on its own stream (P L269 §2.2, P L504 §4.2)."""

    def __init__(self, ppg, dist):
        import torch
        self.ppg = ppg
        self.groups = [dist.new_group(backend="nccl") for _ in range(ppg)]
        self.streams = [torch.cuda.Stream() for _ in range(ppg)]

    def run(self, buf, dist):
        import torch
        cur = torch.cuda.current_stream()
        n = buf.numel()
        q = 4  # slice boundaries on 16 B for fp32/int32 (8 for bf16 is also fine)
        for i, (g, st) in enumerate(zip(self.groups, self.streams)):
            a = (n * i // self.ppg) // q * q
            b = n if i == self.ppg - 1 else (n * (i + 1) // self.ppg) // q * q
            st.wait_stream(cur)
            with torch.cuda.stream(st):
                dist.all_reduce(buf[a:b], group=g)
        for st in self.streams:
            cur.wait_stream(st)


def nccl_ppg(inp, S, P, args, dist, stream, ppg_obj):
    import torch
    buf = inp.clone()
    ms = max_over_ranks(device_time_ms(lambda: ppg_obj.run(buf, dist), args.steps, args.warmup, stream,
                                       lambda: dist.barrier()))
    return {"value": round(busbw(S, P, ms), 2), "unit": "GB/s", "ms_per_step": round(ms, 4),
            "ppg": ppg_obj.ppg, "algo": os.environ.get("NCCL_ALGO", "default")}


def nccl_ring(inp, S, P, args, dist, stream):
    import torch
    buf = inp.clone()
    step = lambda: dist.all_reduce(buf)  # noqa: E731
    ms = max_over_ranks(device_time_ms(step, args.steps, args.warmup, stream, lambda: dist.barrier()))
    return {"value": round(busbw(S, P, ms), 2), "unit": "GB/s", "ms_per_step": round(ms, 4),
            "algo": os.environ.get("NCCL_ALGO", "default"), "version": ".".join(map(str, torch.cuda.nccl.version()))}


def run_sweep(args):
    """busbw vs message size, 1 MiB .. args.mib per rank, ours vs NCCL ring
    (BASELINE metric x-axis). One JSON object per size to args.sweep."""
    import torch
    import torch.distributed as dist
    import paper_2508_13397_b200 as lane
    from seeded_inputs import device as sdev
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("cpu:gloo,cuda:nccl")
    N, G = layout_for(args, world)
    P, dtype, isz = world, args.dtype, itemsize(args.dtype)
    comm = lane.LaneComm(N, G, args.k, rank=rank, device=local)
    stream = torch.cuda.current_stream()
    ppg = NcclPPG(args.nccl_ppg, dist) if args.nccl_ppg > 1 else None
    mib = 1
    rows = []
    while mib <= args.mib:
        n = (mib << 20) // isz
        S = n * isz
        inp = sdev.fill(torch.empty(n, dtype=getattr(torch, dtype), device="cuda"), dtype, "signed", 42, rank)
        out = torch.empty_like(inp)
        regs = []
        if not args.no_register:
            regs = [comm.register(inp), comm.register(out)]
        steps = max(5, min(200, int(2000 / mib)))
        ms = device_time_ms(lambda: comm.allreduce(out, inp), steps, 5, stream, lambda: dist.barrier())
        ok = sample_check([out], N, G, dtype, n, 42, [rank])
        buf = inp.clone()
        ms_n = device_time_ms(lambda: dist.all_reduce(buf), steps, 5, stream, lambda: dist.barrier())
        ms_p = device_time_ms(lambda: ppg.run(buf, dist), steps, 5, stream, lambda: dist.barrier()) if ppg else 0.0
        ms_r, ok_r = 0.0, True
        if args.ring:  # Alg. 1 ring on the same comm (standard approach with k slices)
            ms_r = device_time_ms(lambda: comm.allreduce_ring(out, inp), steps, 5, stream, lambda: dist.barrier())
            ok_r = ring_check(out, P, args.k, dtype, n, 42, comm.plan(n, dtype, algorithm="ring"))
            ok = ok and ok_r
        ms_a = 0.0
        if args.approach2:  # P L296-297; same bits as the lane method
            ms_a = device_time_ms(lambda: comm.allreduce_approach2(out, inp), steps, 5, stream, lambda: dist.barrier())
            ok = ok and sample_check([out], N, G, dtype, n, 42, [rank])
        t = torch.tensor([ms, ms_n, 0.0 if ok else 1.0, ms_p, ms_r, ms_a], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        row = {"layout": f"{N}x{G}", "k": args.k, "dtype": dtype, "bytes": S, "ms": round(t[0].item(), 4),
               "busbw": round(busbw(S, P, t[0].item()), 2), "nccl_ring_ms": round(t[1].item(), 4),
               "nccl_ring_busbw": round(busbw(S, P, t[1].item()), 2), "verified": t[2].item() == 0,
               "frac_of_770": round(busbw(S, P, t[0].item()) / NVLINK_PEAK, 4), "plan": comm.plan(n, dtype)}
        if args.ring:
            row["lane_ring_alg1_busbw"] = round(busbw(S, P, t[4].item()), 2)
            row["lane_ring_alg1_ms"] = round(t[4].item(), 4)
        if args.approach2:
            row["approach2_busbw"] = round(busbw(S, P, t[5].item()), 2)
        row["protocol"] = comm.protocol(n, dtype)
        if ppg:
            row["nccl_ring_ppg"] = args.nccl_ppg
            row["nccl_ring_ppg_busbw"] = round(busbw(S, P, t[3].item()), 2)
        row["registered_buffers"] = bool(regs)
        rows.append(row)
        if rank == 0:
            print(json.dumps(row), flush=True)
        torch.cuda.synchronize()
        dist.barrier()
        for r_ in regs:
            comm.deregister(r_)
        del inp, out, buf
        mib *= 2
    if rank == 0:
        with open(args.sweep, "a") as f:
            for r in rows:
                f.write(json.dumps(r) + "\n")
    comm.close()
    dist.barrier()
    dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.sweep:
        return run_sweep(args)
    if args.impl == "reference":
        return run_reference(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        return run_multi(args)
    if args.gpus > 1:
        raise SystemExit("--gpus > 1 must be launched with torchrun (one process per GPU)")
    return run_single(args)


if __name__ == "__main__":
    sys.exit(main())
