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
N > 1: one process per GPU, real IPC/NVLink; default layout 2 x (N/2)
virtual nodes (8 GPUs: 2 x 4 = configs[1]), k = 1, fp32, 1 GiB per rank.
Bound: NVLink. Without torchrun, ``--gpus N`` launches the N ranks itself
(torch.distributed.run, 127.0.0.1) and relays rank 0's line.

One JSON line is printed by rank 0. Each timed step is one lane_allreduce call
(one kernel launch per round; one round at these sizes) on inputs already in
HBM; inputs are 1 GiB per rank (> 126 MB L2), so no L2 flush is needed.
After the timed region the WHOLE output buffer of every rank is verified on
the device, bit for bit, against the canonical-order sum (DESIGN R#7/R#8) of
the regenerated inputs (plain torch ops here; bench.py never imports oracle/
outside the cpu_baseline leg and the reference arm); value is null on any
mismatch.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# NCCL is used ONLY for the timed comparators (NCCL_ALGO=Ring is the required
# one; the default algorithm is measured on its own communicator as context).
os.environ.setdefault("NCCL_ALGO", "Ring")
# NCCL's version banner goes to stdout; the contract is ONE JSON line from rank 0
if os.environ.get("NCCL_DEBUG", "").upper() in ("VERSION", "WARN"):
    os.environ.pop("NCCL_DEBUG")

METRIC = "allreduce bus GB/s vs msg size at 2/4/8 B200 vs NCCL ring; % of NVLink roofline"
NVLINK_PEAK = 770.0  # GB/s per direction per GPU, measured peer copy (B200_PROFILING.md)
NVLINK_NOMINAL = 900.0
TDT = {"int32": "int32", "float32": "float32", "bfloat16": "bfloat16"}
SHORT = {"int32": "i32", "float32": "f32", "bfloat16": "bf16"}
NVLINK_COUNTERS_NOTE = ("NVLink throughput counters are closed on this pool: `nvidia-smi nvlink -gt d` prints "
                        "'Data Tx: N/A' for every link and NVML NVLINK_THROUGHPUT_DATA_TX/RX answer NOT_SUPPORTED "
                        "(profiles/r02_nvlink_counters.txt); ncu cannot wrap a multi-rank run")


def parse(argv=None):
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
    ap.add_argument("--no-staged", action="store_true",
                    help="multi-GPU: skip timing the unregistered (staged) call beside the registered one")
    ap.add_argument("--nccl-ppg", type=int, default=4,
                    help="multi-GPU: also time the paper's multi-PPG CCL variant (P L269, L504): this many "
                         "NCCL communicators, each allreducing a 1/PPG slice on its own stream (0 = skip)")
    ap.add_argument("--no-register", action="store_true",
                    help="multi-GPU: do not register the buffers (staged path through library scratch)")
    ap.add_argument("--ring", action="store_true",
                    help="sweep: also time the library's ring allreduce (Alg. 1, the paper's standard algorithm)")
    ap.add_argument("--approach2", action="store_true",
                    help="sweep: also time the paper's draft 'approach 2' (node allreduce + lane allreduce)")
    ap.add_argument("--sweep", default=None,
                    help="multi-GPU: write busbw vs message size (ours and NCCL ring) as JSONL to this file")
    ap.add_argument("--sizes", default=None, help="sweep: comma-separated MiB per rank (default 1, 2, 4 .. --mib)")
    ap.add_argument("--repeats", type=int, default=3, help="sweep: timed repeats per cell (median/min/max)")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU test of the launch path: ranks rendezvous over gloo and rank 0 prints a line "
                         "without touching a GPU")
    return ap.parse_args(argv)


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
    """SM clock and throttle-reason sampler running while the timed region
    runs: an NVML thread (5 ms period; the GPU-side work is asynchronous, so
    the sampling thread only competes with the host's launch loop), or the
    nvidia-smi CSV loop where NVML is unavailable. __enter__ returns once the
    first sample is in, so even a short timed region is covered."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpus, period=0.005):
        self.gpus = gpus
        self.period = period
        self.proc = None
        self.thread = None
        self.samples = []  # (sm_mhz, max_mhz, reasons)
        self.source = None
        self.out = os.path.join("/tmp", f"lane_clocks_{os.getpid()}_{id(self)}.csv")

    def _nvml_loop(self, handles, pynvml):
        bits = {"hw_slowdown": pynvml.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": pynvml.nvmlClocksEventReasonSwPowerCap}
        while not self._stop:
            for h in handles:
                try:
                    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
                    r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.samples.append((float(sm), float(mx), {n for n, b in bits.items() if r & b}))
                except Exception:
                    pass
            time.sleep(self.period)

    def __enter__(self):
        import threading
        self._stop = False
        try:
            import pynvml
            pynvml.nvmlInit()
            handles = [pynvml.nvmlDeviceGetHandleByIndex(g) for g in self.gpus]
            self.thread = threading.Thread(target=self._nvml_loop, args=(handles, pynvml), daemon=True)
            self.thread.start()
            self.source = "nvml"
        except Exception:
            self.thread = None
            try:
                self.f = open(self.out, "w")
                self.proc = subprocess.Popen(
                    ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "50",
                     "-i", ",".join(str(g) for g in self.gpus)], stdout=self.f, stderr=subprocess.DEVNULL)
                self.source = "nvidia-smi"
            except Exception:
                self.proc = None
        t0 = time.time()
        while time.time() - t0 < 5.0 and not self._have_sample():
            time.sleep(0.01)
        return self

    def _have_sample(self):
        if self.thread is not None:
            return bool(self.samples)
        if self.proc is None:
            return True
        try:
            return os.path.getsize(self.out) > 0
        except OSError:
            return False

    def __exit__(self, *a):
        self._stop = True
        if self.thread is not None:
            self.thread.join()
        if self.proc:
            self.proc.terminate()
            self.proc.wait()
            self.f.close()

    def summary(self):
        sm, mx, reasons = [], [], set()
        if self.thread is not None:
            for a, b, r in self.samples:
                sm.append(a)
                mx.append(b)
                reasons |= r
        else:
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
                    for nm, v in zip(self.NAMES, f[4:8]):
                        if v.lower().startswith("active"):
                            reasons.add(nm)
            except OSError:
                pass
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0, "source": self.source}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "sm_min_mhz": min(sm),
                "reasons": sorted(reasons), "samples": len(sm), "source": self.source}


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
    """DRAM bytes per launch from the committed ncu `--set full` summary of
    exactly this workload (profiles/*ncu*summary.json: same layout, k, dtype
    and bytes per rank), or (None, None)."""
    import glob
    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", "*ncu*summary.json")), reverse=True):
        try:
            d = json.load(open(f))
        except (OSError, ValueError):
            continue
        w = d.get("workload", "")
        names = {dtype, SHORT[dtype], "fp32" if dtype == "float32" else dtype}
        if not (w.startswith(layout + " ") and f"k={k}" in w and any(nm in w for nm in names)):
            continue
        if d.get("bytes_per_rank") != S:
            continue
        kern = [x for x in d.get("kernels", []) if "lane_tma" in x.get("kernel", "")]
        if not kern or "dram_bytes_per_rank_per_byte" not in kern[0]:
            continue
        return int(kern[0]["dram_bytes_per_rank_per_byte"] * S * P), os.path.basename(f)
    return None, None


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline(N, G, k, dtype, sizes_mib=(1, 16, 64), reps=5):
    """the oracle as it stands (numpy, no tuning) on ONE host
    core of this box (os.sched_setaffinity to the first allowed core,
    OMP/BLAS threads irrelevant: elementwise numpy), layout N x G, k, dtype,
    seed 42; median of `reps` runs at each of 1, 16 and 64 MiB per simulated
    rank. value = busbw at 1 MiB (the CPU-oracle config); the other sizes
    show its scaling."""
    import oracle
    import seeded_inputs as si
    P = N * G
    old_aff = None
    core = None
    try:
        old_aff = os.sched_getaffinity(0)
        core = min(old_aff)
        os.sched_setaffinity(0, {core})
    except (AttributeError, OSError):
        pass
    rows = []
    try:
        for mib in sizes_mib:
            n = (mib << 20) // itemsize(dtype)
            xs = si.generate_all(dtype, "signed", 42, P, n)
            ts = []
            for _ in range(reps):
                t0 = time.perf_counter()
                oracle.lane_allreduce(xs, N, G, k, dtype)
                ts.append(time.perf_counter() - t0)
            del xs
            med = statistics.median(ts)
            rows.append({"mib_per_rank": mib, "median_s": round(med, 4), "min_s": round(min(ts), 4),
                         "max_s": round(max(ts), 4), "busbw": round(busbw(mib << 20, P, med * 1e3), 4)})
    finally:
        if old_aff is not None:
            os.sched_setaffinity(0, old_aff)
    return {"value": rows[0]["busbw"], "unit": "GB/s", "cores": 1, "kind": "oracle",
            "host_cores": os.cpu_count(), "cpu_model": cpu_model(), "pinned_core": core,
            "sample": f"{N}x{G} k={k} {dtype} seed 42, {sizes_mib[0]} MiB per simulated rank ({P} ranks), "
                      f"median of {reps} oracle allreduces on 1 pinned core (numpy); value = busbw at "
                      f"{sizes_mib[0]} MiB; 'sizes' adds {', '.join(str(m) for m in sizes_mib[1:])} MiB",
            "sizes": rows}


# ----------------------------------------------------------------- verification
# bench.py checks its own outputs without the oracle (only the cpu_baseline leg
# and the reference arm run oracle/): the canonical reduction order written out
# here (DESIGN R#7, R#8), once on numpy for sampled positions and once with
# plain torch ops for whole buffers on the device. tests/test_bench_cpu.py pins
# both to the oracle bit for bit.
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


def canonical_lane_sum_torch(xs, N, G, dtype):
    """canonical_lane_sum with plain torch ops on torch tensors (any device):
    fp32 adds in the canonical order (torch's elementwise add is one IEEE
    round-to-nearest add per element), bf16 narrowed with torch's RNE
    conversion once per phase, int32 summed in int64 and wrapped mod 2^32."""
    import torch
    if dtype == "int32":
        acc = xs[0].to(torch.int64)
        for x in xs[1:]:
            acc += x
        acc &= 0xFFFFFFFF
        return torch.where(acc >= 2 ** 31, acc - 2 ** 32, acc).to(torch.int32)
    node = []
    for a in range(N):
        acc = xs[a * G].to(torch.float32, copy=True)
        for h in range(1, G):
            acc += xs[a * G + h].to(torch.float32)
        node.append(acc.to(torch.bfloat16).to(torch.float32) if dtype == "bfloat16" else acc)
    acc = node[0].clone()
    for a in range(1, N):
        acc += node[a]
    return acc.to(torch.bfloat16) if dtype == "bfloat16" else acc


def _bitview(t):
    import torch
    return t.view(torch.int16) if t.element_size() == 2 else t.view(torch.int32)


def verify_whole(outs, N, G, dtype, n, seed, chunk=1 << 24, gen=None):
    """Every element of every tensor in `outs` (all hold the allreduce of the
    P seeded inputs) bit-exact against canonical_lane_sum_torch of the inputs
    regenerated chunk by chunk — on the device by seeded_inputs' CUDA
    generator, or by gen(p, start, m) (CPU tests). Returns (mismatching
    elements, elements checked)."""
    import torch
    P = N * G
    dev = outs[0].device
    tdt = outs[0].dtype
    if gen is None:
        from seeded_inputs import device as sdev

        def gen(p, s, m):
            return sdev.fill(torch.empty(m, dtype=tdt, device=dev), dtype, "signed", seed, p, start=s)
    bad = torch.zeros((), dtype=torch.int64, device=dev)
    for s in range(0, n, chunk):
        m = min(chunk, n - s)
        xs = [gen(p, s, m) for p in range(P)]
        ref = _bitview(canonical_lane_sum_torch(xs, N, G, dtype))
        for o in outs:
            bad += (_bitview(o[s:s + m]) != ref).sum()
        del xs, ref
    if dev.type == "cuda":
        torch.cuda.synchronize()
    return int(bad.item()), n * len(outs)


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


def check_outputs(outs, N, G, dtype, n, seed):
    """Whole-buffer device check (bit-exact) of the direct lane method; the
    ring inter-node stage (LANE_PHASE2=ring) falls back to sample_check.
    Returns {"verified": bool, "elements": checked, "mismatches": m, "how": ...}."""
    if os.environ.get("LANE_PHASE2") == "ring" and N > 2:
        ok = sample_check(outs, N, G, dtype, n, seed, None)
        return {"verified": ok, "elements": None, "mismatches": None,
                "how": "LANE_PHASE2=ring: sampled, exact int / fp within tolerance"}
    bad, checked = verify_whole(outs, N, G, dtype, n, seed)
    return {"verified": bad == 0, "elements": checked, "mismatches": bad,
            "how": "whole buffer, bit-exact vs the canonical-order sum of the regenerated inputs (on device)"}


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
                                  "host_cores": os.cpu_count(), "cpu_model": cpu_model(),
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


# ----------------------------------------------------------------- self-launch
def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def self_launch(args, argv):
    """`python bench.py --gpus N` without torchrun: launch the N ranks the way
    the driver does (torch.distributed.run, one process per GPU, 127.0.0.1),
    pass rank 0's JSON line through (marked), and return the launcher's exit
    code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + list(argv)
    r = subprocess.run(cmd, stdout=subprocess.PIPE, text=True, cwd=ROOT)
    printed = 0
    for line in r.stdout.splitlines():
        try:
            d = json.loads(line)
        except ValueError:
            sys.stderr.write(line + "\n")
            continue
        if isinstance(d, dict) and "metric" in d:
            d["launcher"] = "bench.py self-launch (torch.distributed.run, one process per GPU)"
            print(json.dumps(d), flush=True)
            printed += 1
    if r.returncode == 0 and printed != 1:
        sys.stderr.write(f"bench.py: expected one JSON line from rank 0, got {printed}\n")
        return 1
    return r.returncode


def run_dry(args):
    """--dry-run: the N > 1 plumbing without a GPU (CPU gloo test): rendezvous,
    the max-over-ranks reduction and rank 0's single line."""
    import torch.distributed as dist
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo")
    N, G = layout_for(args, world)
    ms = max_over_ranks(1.0 + rank)
    if rank == 0:
        line = base_line(args, world, args.steps, args.warmup)
        line.update({"value": None, "ms_per_step": ms, "dry_run": True,
                     "config": {"workload": f"dry run {N}x{G}", "layout": f"{N}x{G}", "world": world}})
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0


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
    chk = check_outputs(outs, N, G, dtype, n, seed)
    ok = chk["verified"]
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
        "verified": ok, "verification": chk,
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
        line["cpu_baseline"] = cpu_baseline(N, G, k, dtype)
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
    ok = all(torch.equal(_bitview(h), _bitview(outs[0].cpu())) for h in h_out[:1])
    return {"value": round(busbw(S, P, ms), 2) if ok else None, "unit": "GB/s", "ms_per_step": round(ms, 3),
            "h2d_bytes_per_step": P * S, "d2h_bytes_per_step": P * S, "verified": ok,
            "api": "lane_allreduce_emulated_host (C ABI, pinned host buffers)"}


# ----------------------------------------------------------------- N > 1
def nccl_default_group(dist):
    """A communicator created with NCCL_ALGO unset: NCCL's own algorithm
    choice (NVLS / tree / ring), measured as labelled context only. NCCL reads
    NCCL_ALGO when a communicator is created; torch creates it at the group's
    first collective, done here with the variable removed."""
    import torch
    old = os.environ.pop("NCCL_ALGO", None)
    try:
        g = dist.new_group(backend="nccl")
        t = torch.zeros(1024, device="cuda")
        dist.all_reduce(t, group=g)
        torch.cuda.synchronize()
    finally:
        if old is not None:
            os.environ["NCCL_ALGO"] = old
    return g


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
    barrier = lambda: dist.barrier()  # noqa: E731
    # the comparators' communicators first: NCCL_ALGO=Ring on the default group,
    # then NCCL's default algorithm on its own group (context)
    if not args.no_nccl:
        t = torch.zeros(1024, device="cuda")
        dist.all_reduce(t)
        g_default = nccl_default_group(dist)
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
    step = lambda: comm.allreduce(out, inp)  # noqa: E731
    clk = Clocks(list(range(world))) if rank == 0 else None
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if clk:
        clk.__enter__()
    ms = device_time_ms(step, args.steps, 0, stream, barrier)
    if clk:
        clk.__exit__()
    comm.check()
    ms_max = max_over_ranks(ms)
    chk = check_outputs([out], N, G, dtype, n, seed)
    agg = torch.tensor([0 if chk["verified"] else 1, chk["elements"] or 0], dtype=torch.int64)
    dist.all_reduce(agg)
    ok = int(agg[0]) == 0
    chk = dict(chk, verified=ok, elements=int(agg[1]) if chk["elements"] is not None else None,
               mismatching_ranks=int(agg[0]))
    bw = busbw(S, P, ms_max)
    launches = max(plan["launches"], 1)
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
        "verified": ok, "verification": chk,
        "roofline": {"bound": "nvlink", "achieved": round(bw, 2), "peak": NVLINK_PEAK, "unit": "GB/s",
                     "frac": round(bw / NVLINK_PEAK, 4), "frac_of_nominal_900": round(bw / NVLINK_NOMINAL, 4),
                     "traffic": None, "traffic_note": NVLINK_COUNTERS_NOTE,
                     "peak_source": "measured peer copy per direction, B200_PROFILING.md (no NVLink entry in "
                                    "MEASURED_PEAKS.json)",
                     "algorithmic_bytes_per_launch": int(2 * (P - 1) / P * S / launches),
                     "algorithmic_basis": "NVLink bytes out of (= into) each GPU per launch: 2(P-1)/P S"},
        "gpu_launches": args.steps * launches,
    })
    if clk:
        line["clocks"] = clk.summary()
    if registered and not args.no_staged:
        line["staged"] = staged_multi(comm, inp, N, G, dtype, n, S, args, dist, stream)
    if not args.no_e2e:
        line["e2e"] = e2e_multi(comm, inp, N, G, dtype, n, S, args, dist)
    if not args.no_nccl:
        line["nccl_ring"] = nccl_ring(inp, S, P, args, dist, stream)
        if args.nccl_ppg > 1:
            line["nccl_ring_multi_ppg"] = nccl_ppg(inp, S, P, args, dist, stream, NcclPPG(args.nccl_ppg, dist))
        line["nccl_default_context"] = nccl_ring(inp, S, P, args, dist, stream, group=g_default,
                                                 algo="default (NCCL_ALGO unset; context only)")
    if rank == 0 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(N, G, k, dtype)
    dist.barrier()
    if rank == 0:
        print(json.dumps(line), flush=True)
    comm.close()
    dist.barrier()
    dist.destroy_process_group()
    return 0 if ok else 1


def staged_multi(comm, inp, N, G, dtype, n, S, args, dist, stream):
    """The path a plain lane_allreduce caller gets: unregistered buffers,
    staged through the library's scratch (DESIGN §6 job set 'staged')."""
    import torch
    si_ = inp.clone()
    so_ = torch.empty_like(si_)
    ms = max_over_ranks(device_time_ms(lambda: comm.allreduce(so_, si_), args.steps, args.warmup, stream,
                                       lambda: dist.barrier()))
    comm.check()
    chk = check_outputs([so_], N, G, dtype, n, 42)
    okt = torch.tensor([0 if chk["verified"] else 1])
    dist.all_reduce(okt)
    ok = okt.item() == 0
    P = N * G
    del si_, so_
    return {"value": round(busbw(S, P, ms), 2) if ok else None, "unit": "GB/s", "ms_per_step": round(ms, 4),
            "verified": ok, "registered_buffers": False, "job_set": "staged (library scratch)"}


def e2e_multi(comm, inp, N, G, dtype, n, S, args, dist):
    import torch
    # 2 x S of pinned host memory per rank (16 GiB at 8 ranks x 1 GiB): every
    # rank allocates first and the ranks agree before any collective timing,
    # so one rank short of pinned memory cannot leave the others in a barrier
    err = None
    try:
        h_in = torch.empty(n, dtype=inp.dtype).pin_memory()
        h_in.copy_(inp)
        h_out = torch.empty_like(h_in).pin_memory()
    except (RuntimeError, MemoryError) as e:  # pinned allocation failed
        err = str(e).splitlines()[0][:200]
    bad = torch.tensor([0 if err is None else 1])
    dist.all_reduce(bad)
    if int(bad.item()):
        return {"value": None, "unit": "GB/s", "h2d_bytes_per_step": S, "d2h_bytes_per_step": S,
                "error": err or "pinned host allocation failed on another rank"}
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

    def __init__(self, ppg, dist, backend="nccl"):
        import torch
        self.ppg = ppg
        self.groups = [dist.new_group(backend=backend) for _ in range(ppg)]
        self.streams = [torch.cuda.Stream() for _ in range(ppg)] if backend == "nccl" else None

    @staticmethod
    def slices(n, ppg, q=4):
        """[a, b) of every communicator's slice: contiguous, covering [0, n),
        boundaries on q elements (16 B for fp32/int32)."""
        out = []
        for i in range(ppg):
            a = (n * i // ppg) // q * q
            b = n if i == ppg - 1 else (n * (i + 1) // ppg) // q * q
            out.append((a, b))
        return out

    def run(self, buf, dist):
        import torch
        if self.streams is None:  # CPU (gloo) test of the slicing: one communicator after the other
            for (a, b), g in zip(self.slices(buf.numel(), self.ppg), self.groups):
                dist.all_reduce(buf[a:b], group=g)
            return
        cur = torch.cuda.current_stream()
        for (a, b), g, st in zip(self.slices(buf.numel(), self.ppg), self.groups, self.streams):
            st.wait_stream(cur)
            with torch.cuda.stream(st):
                dist.all_reduce(buf[a:b], group=g)
        for st in self.streams:
            cur.wait_stream(st)


def nccl_ppg(inp, S, P, args, dist, stream, ppg_obj):
    buf = inp.clone()
    ms = max_over_ranks(device_time_ms(lambda: ppg_obj.run(buf, dist), args.steps, args.warmup, stream,
                                       lambda: dist.barrier()))
    return {"value": round(busbw(S, P, ms), 2), "unit": "GB/s", "ms_per_step": round(ms, 4),
            "ppg": ppg_obj.ppg, "algo": os.environ.get("NCCL_ALGO", "default")}


def nccl_ring(inp, S, P, args, dist, stream, group=None, algo=None):
    import torch
    buf = inp.clone()
    step = lambda: dist.all_reduce(buf, group=group)  # noqa: E731
    ms = max_over_ranks(device_time_ms(step, args.steps, args.warmup, stream, lambda: dist.barrier()))
    return {"value": round(busbw(S, P, ms), 2), "unit": "GB/s", "ms_per_step": round(ms, 4),
            "algo": algo or os.environ.get("NCCL_ALGO", "default"),
            "version": ".".join(map(str, torch.cuda.nccl.version()))}


def sweep_sizes(args):
    if args.sizes:
        return [float(x) for x in args.sizes.split(",")]
    out, m = [], 1
    while m <= args.mib:
        out.append(float(m))
        m *= 2
    return out


def timed_repeats(fn, steps, warmup, stream, dist, repeats):
    """`repeats` timed runs of `steps` calls (max over ranks each):
    (median, min, max) in ms per call (the paper repeats
    its runs, P L422)."""
    ts = []
    for r in range(repeats):
        ts.append(max_over_ranks(device_time_ms(fn, steps, warmup if r == 0 else 1, stream,
                                                lambda: dist.barrier())))
    return statistics.median(ts), min(ts), max(ts)


def run_sweep(args):
    """busbw vs message size per rank, ours vs NCCL ring (BASELINE metric
    x-axis). Every cell: `--repeats` timed runs (median / min / max, max over
    ranks each) with the nvidia-smi clock record of the cell, and the whole
    output buffer verified on the device. One JSON object per size to
    args.sweep (rank 0)."""
    import torch
    import torch.distributed as dist
    import paper_2508_13397_b200 as lane
    from seeded_inputs import device as sdev
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("cpu:gloo,cuda:nccl")
    t = torch.zeros(1024, device="cuda")
    dist.all_reduce(t)
    g_default = None if args.no_nccl else nccl_default_group(dist)
    N, G = layout_for(args, world)
    P, dtype, isz = world, args.dtype, itemsize(args.dtype)
    comm = lane.LaneComm(N, G, args.k, rank=rank, device=local)
    stream = torch.cuda.current_stream()
    ppg = NcclPPG(args.nccl_ppg, dist) if (args.nccl_ppg > 1 and not args.no_nccl) else None
    rows = []
    R = args.repeats

    def bw(ms):
        return round(busbw(S, P, ms), 2)

    for mib in sweep_sizes(args):
        n = int(mib * (1 << 20)) // isz
        S = n * isz
        inp = sdev.fill(torch.empty(n, dtype=getattr(torch, dtype), device="cuda"), dtype, "signed", 42, rank)
        out = torch.empty_like(inp)
        regs = []
        if not args.no_register:
            regs = [comm.register(inp), comm.register(out)]
        steps = max(5, min(200, int(2000 / mib)))
        clk = Clocks(list(range(world))) if rank == 0 else None
        if clk:
            clk.__enter__()
        ms = timed_repeats(lambda: comm.allreduce(out, inp), steps, 5, stream, dist, R)
        if clk:
            clk.__exit__()
        comm.check()
        chk = check_outputs([out], N, G, dtype, n, 42)
        row = {"layout": f"{N}x{G}", "k": args.k, "dtype": dtype, "bytes": S, "steps": steps, "repeats": R,
               "ms": round(ms[0], 4), "ms_min": round(ms[1], 4), "ms_max": round(ms[2], 4),
               "busbw": bw(ms[0]), "busbw_min": bw(ms[2]), "busbw_max": bw(ms[1]),
               "frac_of_770": round(busbw(S, P, ms[0]) / NVLINK_PEAK, 4), "plan": comm.plan(n, dtype),
               "protocol": comm.protocol(n, dtype), "registered_buffers": bool(regs)}
        ok = chk["verified"]
        if not args.no_nccl:
            buf = inp.clone()
            mn = timed_repeats(lambda: dist.all_reduce(buf), steps, 5, stream, dist, R)
            row.update({"nccl_ring_ms": round(mn[0], 4), "nccl_ring_busbw": bw(mn[0])})
            md = timed_repeats(lambda: dist.all_reduce(buf, group=g_default), steps, 5, stream, dist, R)
            row.update({"nccl_default_busbw": bw(md[0]), "nccl_default_note": "NCCL_ALGO unset; context only"})
            if ppg:
                mp = timed_repeats(lambda: ppg.run(buf, dist), steps, 5, stream, dist, R)
                row.update({"nccl_ring_ppg": args.nccl_ppg, "nccl_ring_ppg_busbw": bw(mp[0])})
            del buf
        if args.ring:  # Alg. 1 ring on the same comm (standard approach with k slices)
            mr = timed_repeats(lambda: comm.allreduce_ring(out, inp), steps, 5, stream, dist, R)
            ok = ok and ring_check(out, P, args.k, dtype, n, 42, comm.plan(n, dtype, algorithm="ring"))
            row.update({"lane_ring_alg1_ms": round(mr[0], 4), "lane_ring_alg1_busbw": bw(mr[0]),
                        "ring_protocol": comm.ring_protocol(n, dtype)})
        if args.approach2:  # P L296-297; same bits as the lane method
            ma = timed_repeats(lambda: comm.allreduce_approach2(out, inp), steps, 5, stream, dist, R)
            ok = ok and check_outputs([out], N, G, dtype, n, 42)["verified"]
            row["approach2_busbw"] = bw(ma[0])
        okt = torch.tensor([0 if ok else 1])
        dist.all_reduce(okt)
        row["verified"] = okt.item() == 0
        row["verified_how"] = chk["how"]
        if clk:
            row["clocks"] = clk.summary()
        rows.append(row)
        if rank == 0:
            print(json.dumps(row), flush=True)
        torch.cuda.synchronize()
        dist.barrier()
        for r_ in regs:
            comm.deregister(r_)
        del inp, out
        torch.cuda.empty_cache()
    if rank == 0:
        with open(args.sweep, "a") as f:
            for r in rows:
                f.write(json.dumps(r) + "\n")
    comm.close()
    dist.barrier()
    dist.destroy_process_group()
    return 0


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    args = parse(argv)
    if args.impl == "reference":
        return run_reference(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus > 1 and world == 1 and "RANK" not in os.environ:
        return self_launch(args, argv)
    if args.dry_run:
        return run_dry(args)
    if args.sweep:
        return run_sweep(args)
    if world > 1:
        return run_multi(args)
    return run_single(args)


if __name__ == "__main__":
    sys.exit(main())
