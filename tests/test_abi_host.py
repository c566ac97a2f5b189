"""Host-only checks of the C-ABI library (``-m "not gpu"``, no GPU needed).

- the library loads and exports every function include/lane_allreduce.h declares;
- the library's own topology and partition (the code the kernels run, via the
  shared lane_plan.h) equal the oracle's, which was written independently;
- argument validation names the offending field;
- the binding fails loudly without the library; the reference arm prints the contract line.
"""
import ctypes
import os

import numpy as np
import pytest

import oracle
from paper_2508_13397_b200 import _lib
import paper_2508_13397_b200 as lane


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    syms = _lib.header_symbols()
    assert len(syms) == 29, syms
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in include/lane_allreduce.h but not exported"
    assert "sm_100a" in lane.version()


@pytest.mark.parametrize("N,G", [(1, 1), (2, 4), (4, 2), (8, 1), (1, 8), (3, 5), (16, 1)])
def test_topology_matches_oracle(N, G):
    t = oracle.Topology(N, G, 1)
    for p in range(N * G):
        node, gpu, grp, ln = lane.topology(N, G, p)
        assert (node, gpu) == (t.node(p), t.gpu(p))
        assert grp == t.comm_group(p)
        assert ln == t.comm_lane(p)


@pytest.mark.parametrize("n,itemsize,N,G,k,cg,rg", [
    (262144, 4, 2, 4, 1, 0, 0), (10, 4, 1, 4, 1, 0, 0), (1, 4, 2, 4, 8, 0, 0),
    (1000003, 4, 4, 2, 4, 4096, 0), (1000003, 2, 8, 1, 8, 999, 70001), (7, 2, 2, 2, 2, 1, 0),
    (64, 4, 1, 8, 8, 0, 0), (0, 4, 2, 2, 2, 0, 0), (4099, 4, 2, 4, 3, 5, 33), (123457, 2, 2, 4, 16, 64, 1000),
    (2 ** 20 + 3, 4, 2, 4, 1, 16384, 2 ** 16)])
def test_partition_matches_oracle(n, itemsize, N, G, k, cg, rg):
    mine = lane.partition_units(n, itemsize, N, G, k, cg, rg)
    ref = oracle.partition(n, itemsize, N, G, k, cg or None, rg or None)
    assert len(mine) == len(ref)
    for m, u in zip(mine, ref):
        assert m == (u.round, u.l, u.c, u.g, u.a, u.part_start, u.part_end, u.start, u.end)


def test_partition_random_matches_oracle():
    rng = np.random.default_rng(5)
    for _ in range(60):
        N, G = int(rng.integers(1, 5)), int(rng.integers(1, 5))
        k = int(rng.integers(1, 17))
        itemsize = int(rng.choice([2, 4]))
        n = int(rng.integers(0, 200000))
        cg = int(rng.choice([0, 1, 7, 64, 1000]))
        rg = int(rng.choice([0, 100, 5000]))
        mine = lane.partition_units(n, itemsize, N, G, k, cg, rg)
        ref = oracle.partition(n, itemsize, N, G, k, cg or None, rg or None)
        assert [m for m in mine] == [(u.round, u.l, u.c, u.g, u.a, u.part_start, u.part_end, u.start, u.end)
                                     for u in ref], (n, itemsize, N, G, k, cg, rg)


def test_validation_names_the_field():
    lib = _lib.load()
    h = ctypes.c_void_p()
    for args, field in (((0, 4, 1, 0, 0), "nodes"), ((2, 0, 1, 0, 0), "gpus_per_node"),
                        ((2, 4, 0, 0, 0), "procs_per_gpu"), ((2, 4, 17, 0, 0), "procs_per_gpu"),
                        ((4, 8, 1, 0, 0), "LANE_MAX_RANKS"), ((2, 4, 1, 8, 0), "rank")):
        code = lib.lane_allreduce_init_rank(*args, ctypes.byref(h))
        assert code == -1
        assert not h.value
        assert field in lib.lane_allreduce_last_error(None).decode()
    assert lib.lane_topology_query(2, 4, 8, None, None, None, None) == -1
    assert lib.lane_partition_query(10, 3, 1, 1, 1, 0, 0, None, 0, None) == -2


def test_missing_library_fails_loudly(monkeypatch):
    """No fallback: without the CUDA library the binding raises (never a CPU path)."""
    import paper_2508_13397_b200 as lane
    monkeypatch.setattr(_lib, "LIB_PATH", os.path.join(os.path.dirname(_lib.LIB_PATH), "absent.so"))
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(ImportError):
        _lib.load()
    with pytest.raises(ImportError):
        lane.LaneEmulator(2, 2, 1, device=0)


def test_reference_arm_line_n1_cpu():
    """``bench.py --impl reference`` at N = 1 prints the contract line on CPU."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "1"], capture_output=True, text=True, timeout=300, cwd=root, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e", "gpu_launches"):
        assert key in d, key
    assert d["impl"] == "reference" and d["n_gpus"] == 1 and d["steps"] == 1 and d["warmup"] == 1
    assert d["unit"] == d["e2e"]["unit"] == "GB/s" and d["higher_is_better"] is True
    assert d["config"]["layout"] == "2x4" and d["cpu_baseline"]["cores"] >= 1
