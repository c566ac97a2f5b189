"""Multi-process host paths on CPU (world size 2, gloo; no GPU).

What of the N > 1 path runs without a GPU: the IPC-handle / registration blob
exchange (``exchange_blobs``, the paper's handle broadcast P L330), the
environment-driven C-ABI init of one process per GPU (``lane_allreduce_init``
reads RANK / LOCAL_RANK / WORLD_SIZE), the bench's max-over-ranks device-time
reduction and virtual layouts, and the reference arm's torchrun contract
(rank 0 alone prints one JSON line, the other ranks exit 0 without work).
"""
import ctypes
import json
import os
import socket
import subprocess
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, fn_name, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    sys.path.insert(0, ROOT)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, globals()[fn_name](rank, world)))
    except Exception as e:  # reported to the parent
        q.put((rank, f"ERROR {type(e).__name__}: {e}"))
    finally:
        dist.destroy_process_group()


def _spawn(fn_name, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, fn_name, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r, v in out.items():
        assert not (isinstance(v, str) and v.startswith("ERROR")), (r, v)
    return out


# ----------------------------------------------------------------- workers
def _exchange(rank, world):
    from paper_2508_13397_b200 import exchange_blobs
    blob = bytes([rank + 1]) * 64 + rank.to_bytes(4, "little")  # fixed size, rank-specific
    got = exchange_blobs(blob)
    return [b.hex() for b in got]


def _init_env(rank, world):
    from paper_2508_13397_b200 import _lib
    lib = _lib.load()
    h = ctypes.c_void_p()
    res = {}
    # nodes*gpus_per_node must equal WORLD_SIZE (2): 2x2 is rejected before any CUDA call
    res["mismatch"] = (lib.lane_allreduce_init(2, 2, 1, ctypes.byref(h)), h.value,
                       lib.lane_allreduce_last_error(None).decode())
    # RANK missing: rejected
    saved = os.environ.pop("RANK")
    res["no_rank"] = (lib.lane_allreduce_init(1, 2, 1, ctypes.byref(h)), h.value,
                      lib.lane_allreduce_last_error(None).decode())
    os.environ["RANK"] = saved
    return res


def _max_over_ranks(rank, world):
    import bench
    return bench.max_over_ranks(1.5 + 2.25 * rank)


def _nccl_ppg_slices(rank, world):
    import torch
    import bench
    ppg = bench.NcclPPG(4, dist, backend="gloo")
    res = {}
    for n in (1, 7, 64, 4099, 100003):
        buf = torch.arange(n, dtype=torch.float32) * (rank + 1)
        ppg.run(buf, dist)
        want = torch.arange(n, dtype=torch.float32) * sum(r + 1 for r in range(world))
        res[n] = bool(torch.equal(buf, want))
    return res


# ----------------------------------------------------------------- tests
def test_nccl_ppg_comparator_slices():
    """The multi-PPG CCL comparator (P L269, L504): PPG
    communicators each allreduce one slice; the slices are contiguous, cover
    the buffer exactly with 16-byte boundaries, and together give the full
    allreduce (gloo stand-in for NCCL, world size 2)."""
    import bench
    for n in (0, 1, 7, 64, 4099, 1 << 20):
        for ppg in (1, 2, 4, 16):
            sl = bench.NcclPPG.slices(n, ppg)
            assert sl[0][0] == 0 and sl[-1][1] == n
            assert all(b0 == a1 for (_, b0), (a1, _) in zip(sl, sl[1:]))
            assert all(a % 4 == 0 for a, _ in sl)
    out = _spawn("_nccl_ppg_slices")
    assert all(all(v.values()) for v in out.values()), out


def test_exchange_blobs_rank_order_gloo():
    out = _spawn("_exchange")
    want = [(bytes([r + 1]) * 64 + r.to_bytes(4, "little")).hex() for r in range(2)]
    assert out[0] == want and out[1] == want


def test_env_init_validates_world_size_gloo():
    out = _spawn("_init_env")
    for r in range(2):
        code, h, msg = out[r]["mismatch"]
        assert code == -1 and not h and "WORLD_SIZE" in msg
        code, h, msg = out[r]["no_rank"]
        assert code == -1 and not h and "RANK" in msg


def test_bench_max_over_ranks_gloo():
    out = _spawn("_max_over_ranks")
    assert out[0] == out[1] == 3.75  # the slowest rank's device time, on every rank


def test_bench_layouts():
    sys.path.insert(0, ROOT)
    import bench

    class A:
        layout = None
    assert [bench.layout_for(A, P) for P in (1, 2, 4, 8)] == [(2, 4), (2, 1), (2, 2), (2, 4)]
    assert bench.layout_for(A, 3) == (3, 1)
    A.layout = "4x2"
    assert bench.layout_for(A, 8) == (4, 2)


def test_reference_arm_under_torchrun_cpu():
    """``bench.py --impl reference`` launched as the driver launches N > 1:
    rank 0 prints exactly one JSON line (impl reference, the oracle timed on
    host cores), rank 1 prints nothing; both exit 0."""
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "1"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT,
                       env={**os.environ, "OMP_NUM_THREADS": "1"})
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["config"]["layout"] == "2x1"


@pytest.mark.parametrize("gpus", [2, 4, 8])
def test_bench_self_launch_without_torchrun_cpu(gpus):
    """``python bench.py --gpus N`` WITHOUT torchrun (no RANK / WORLD_SIZE):
    bench.py launches the N ranks itself through torch.distributed.run on
    127.0.0.1 and relays rank 0's single JSON line (the --dry-run path does
    the rendezvous and the max-over-ranks reduction without a GPU)."""
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR",
                                                            "MASTER_PORT")}
    env["OMP_NUM_THREADS"] = "1"
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(gpus), "--dry-run", "--steps", "2",
           "--warmup", "3"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == gpus and d["dry_run"] and d["ms_per_step"] == float(gpus)  # max over ranks of 1 + rank
    assert d["launcher"].startswith("bench.py self-launch")
    assert d["config"]["layout"] == f"2x{gpus // 2}"
