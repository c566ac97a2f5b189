"""Multi-GPU parity (``-m gpu``): torchrun one process per GPU over NVLink.

Skipped when the box has fewer GPUs than the world size under test."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus():
    import torch
    return torch.cuda.device_count()


@pytest.mark.parametrize("P", [2, 4, 8])
def test_multigpu_parity(P):
    if _ngpus() < P:
        pytest.skip(f"needs {P} GPUs, have {_ngpus()}")
    port = 29500 + P
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={P}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "tests", "mp_worker.py"), "--quick"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert f"mp_worker P={P}: OK" in out, out[-4000:]


def test_watchdog_timeout_p2():
    """A call that a peer never joins ends by the device watchdog
    (LANE_ERR_TIMEOUT) instead of hanging the GPU (simple and LL protocols)."""
    if _ngpus() < 2:
        pytest.skip("needs 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29611",
           os.path.join(ROOT, "tests", "mp_timeout_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "mp_timeout_worker: OK" in out, out[-4000:]


@pytest.mark.parametrize("P", [2, 4, 8])
def test_stress_back_to_back(P):
    """Back-to-back calls on one comm per virtual layout (every layout of P)
    across the LL / LL128 / simple / bulk-store thresholds, int32 / fp32 / bf16,
    registered or not, in place or not; every call checked bit-exactly
    (fp32 / bf16 included: R#25, the LL128 line property, at up to 7 writers
    per GPU through NVSwitch when P = 8). Budget: P = 4 ran 3 layouts x 20000
    calls in about 20 s (profiles/r02_stress_final.txt); every P runs 3000 per layout."""
    if _ngpus() < P:
        pytest.skip(f"needs {P} GPUs, have {_ngpus()}")
    iters = 3000
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={P}",
           "--master-addr", "127.0.0.1", "--master-port", str(29620 + P),
           os.path.join(ROOT, "tests", "mp_stress_worker.py"), "--iters", str(iters), "--layouts", "all"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200, cwd=ROOT)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "mp_stress_worker" in out and ": OK" in out, out[-4000:]
