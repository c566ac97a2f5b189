"""Per-CTA stall accounting of one lane allreduce launch (LANE_TRACE=1).

torchrun --nproc-per-node P tools/trace_run.py --layout 2x1 [--k 1] [--mib 1024]
python tools/trace_run.py --emulated --layout 2x4
Prints, per rank, the mean / max over CTAs of every trace field in microseconds.
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["LANE_TRACE"] = "1"

import torch  # noqa: E402

import paper_2508_13397_b200 as lane  # noqa: E402
from seeded_inputs import device as sdev  # noqa: E402


def summarize_ll(tr, label):
    """LL kernel trace: words 0..5 = CTA start, last thread's end of phase A..E."""
    keys = lane.LaneComm.TRACE_FIELDS[:6]
    rows = [[t[k] for k in keys] for t in tr if t[keys[0]]]
    t0 = min(r[0] for r in rows)
    out = [label + f"  (LL protocol, {len(rows)} CTAs; us after the first CTA started)"]
    out.append(f"  CTA start        min {0:9.2f}  max {(max(r[0] for r in rows) - t0) / 1e3:9.2f}")
    ent = [t["entry_abs"] for t in tr if t.get("entry_abs")]
    if ent:  # before the PDL wait: how early the CTAs were resident
        out.append(f"  CTA entry (pre-PDL-wait) min {(min(ent) - t0) / 1e3:9.2f}  max {(max(ent) - t0) / 1e3:9.2f}")
    for i, ph in enumerate("ABCDE", start=1):
        v = [r[i] for r in rows if r[i]]
        if v:
            out.append(f"  end of phase {ph}   min {(min(v) - t0) / 1e3:9.2f}  max {(max(v) - t0) / 1e3:9.2f}")
    return "\n".join(out)


def smid_report(tr, label, key):
    """Does a CTA's time to finish `key` follow the SM it ran on? Mean per SM
    class (smid halves, parity, TPC pairs) and the SMs of the 12 slowest and
    fastest CTAs."""
    rows = [(t["smid"], t[key]) for t in tr if t.get(key)]
    if not rows:
        return ""
    vals = sorted(rows, key=lambda r: r[1])
    m = statistics.mean(v for _, v in rows)

    def cls(name, f):
        a = [v for s, v in rows if f(s)]
        b = [v for s, v in rows if not f(s)]
        return f"{name}: {statistics.mean(a) / m:.3f} vs {statistics.mean(b) / m:.3f}" if a and b else ""
    out = [f"  {label} {key}: per-SM classes (mean / overall mean): " +
           "; ".join(x for x in (cls("smid<74", lambda s: s < 74), cls("even smid", lambda s: s % 2 == 0),
                                 cls("smid%4<2", lambda s: s % 4 < 2), cls("smid%16<8", lambda s: s % 16 < 8)) if x)]
    out.append("  slowest SMs: " + " ".join(str(s) for s, _ in vals[-12:][::-1]))
    out.append("  fastest SMs: " + " ".join(str(s) for s, _ in vals[:12]))
    return "\n".join(out)


def dump(tr, ll, path):
    with open(path, "a") as f:
        for i, t in enumerate(tr):
            f.write(json.dumps(dict(t, cta=i, ll=ll)) + "\n")


def summarize(tr, label):
    keys = lane.LaneComm.TRACE_FIELDS
    out = [label]
    st = [t["start_abs"] for t in tr if t["start_abs"]]
    ends = [t["end_abs"] for t in tr if t["end_abs"]]
    if st:
        out.append(f"  CTA start spread {(max(st) - min(st)) / 1e3:9.2f} us; end-of-call barrier passed at "
                   f"{(max(ends) - min(st)) / 1e3 if ends else float('nan'):9.2f} us after the first CTA start")
    for key in keys:
        if key in ("start_abs", "end_abs"):
            continue
        v = [t[key] for t in tr]
        if key in ("prod_tiles", "store_jobs", "bytes_stored"):
            out.append(f"  {key:16s} mean {statistics.mean(v):12.1f}  max {max(v):12.1f}")
        else:
            out.append(f"  {key:16s} mean {statistics.mean(v) / 1e3:9.1f} us  max {max(v) / 1e3:9.1f} us")
    return "\n".join(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layout", default="2x1")
    ap.add_argument("--k", type=int, default=1)
    ap.add_argument("--mib", type=float, default=1024)
    ap.add_argument("--dtype", default="float32")
    ap.add_argument("--emulated", action="store_true")
    ap.add_argument("--register", action="store_true", help="register the buffers (direct-push job set, as bench.py)")
    ap.add_argument("--dump", default=None, help="append every CTA's trace record (JSON lines) to this file")
    ap.add_argument("--calls", type=int, default=1,
                    help="back-to-back calls before reading the trace (>1: steady state, no launch skew)")
    a = ap.parse_args()
    N, G = map(int, a.layout.split("x"))
    tdt = getattr(torch, a.dtype)
    n = int(a.mib * (1 << 20)) // (2 if a.dtype == "bfloat16" else 4)
    if a.emulated:
        emu = lane.LaneEmulator(N, G, a.k, device=0)
        ins = [sdev.fill(torch.empty(n, dtype=tdt, device="cuda"), a.dtype, "signed", 1, p) for p in range(N * G)]
        outs = [torch.empty_like(t) for t in ins]
        for _ in range(3):
            emu.allreduce(outs, ins)
        torch.cuda.synchronize()
        summ = summarize_ll if emu.protocol(n, a.dtype) in ("ll", "ll128") else summarize
        print(summ(emu.trace(), f"emulated {a.layout} k={a.k}"), flush=True)
        return
    import torch.distributed as dist
    rank, local = int(os.environ["RANK"]), int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    comm = lane.LaneComm(N, G, a.k, rank=rank, device=local)
    inp = sdev.fill(torch.empty(n, dtype=tdt, device="cuda"), a.dtype, "signed", 1, rank)
    out = torch.empty_like(inp)
    if a.register:
        comm.register(inp)
        comm.register(out)
    for _ in range(3):
        comm.allreduce(out, inp)
    torch.cuda.synchronize()
    dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(a.calls):
        comm.allreduce(out, inp)
    e.record()
    torch.cuda.synchronize()
    tr = comm.trace()
    summ = summarize_ll if comm.protocol(n, a.dtype) in ("ll", "ll128") else summarize
    ll = comm.protocol(n, a.dtype) in ("ll", "ll128")
    txt = summ(tr, f"rank {rank} {a.layout} k={a.k} ctas={len(tr)} kernel {s.elapsed_time(e) / a.calls:.4f} ms/call over {a.calls} calls")
    if ll:  # phase-A end (word 1) relative to the CTA's start (word 0)
        tr2 = [dict(t, a_time=t[lane.LaneComm.TRACE_FIELDS[1]] - t[lane.LaneComm.TRACE_FIELDS[0]]) for t in tr]
        txt += "\n" + smid_report(tr2, f"rank {rank}", "a_time")
    else:
        txt += "\n" + smid_report(tr, f"rank {rank}", "phase_A")
    if a.dump:
        dump(tr, ll, a.dump.replace("%r", str(rank)))
    for r in range(dist.get_world_size()):
        if r == rank:
            print(txt, flush=True)
        dist.barrier()
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
