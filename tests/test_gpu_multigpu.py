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


@pytest.mark.parametrize("P", [2, 4])
def test_ranks_sharing_one_gpu(P):
    """P processes on cuda:0 through the multi-GPU code path (same-device IPC
    peers, system-scope flags, the start handshake and end barrier, staged and
    registered buffers, every layout of P, k = 1 and 2, simple / bulk stores /
    chunk claims / LL / LL128, fp32 / bf16 / int32) bit-exactly against the
    oracle — so a box with ONE GPU runs the IPC path too (their kernels share
    the GPU; every cross-rank wait is bounded by the watchdog). P = 2 about
    10 s, P = 4 about 60 s on a B200 (profiles/r02_samedev.txt)."""
    if _ngpus() < 1:
        pytest.skip("needs a GPU")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={P}",
           "--master-addr", "127.0.0.1", "--master-port", str(29640 + P),
           os.path.join(ROOT, "tests", "mp_samedev_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "mp_samedev_worker: OK" in out, out[-4000:]


def test_watchdog_and_mismatch_sharing_one_gpu():
    """test_watchdog_timeout_p2's cases (watchdog on a call a peer never joins;
    LANE_ERR_MISMATCH from the start handshake) with both ranks on cuda:0."""
    if _ngpus() < 1:
        pytest.skip("needs a GPU")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29651",
           os.path.join(ROOT, "tests", "mp_timeout_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT,
                       env=dict(os.environ, LANE_TEST_DEVICE="0"))
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "mp_timeout_worker: OK" in out, out[-4000:]


@pytest.mark.parametrize("P", [2, 4])
def test_stress_sharing_one_gpu(P):
    """test_stress_back_to_back (every layout of P, every protocol threshold,
    bit-exact per call) with all P ranks on cuda:0, 300 calls per layout."""
    if _ngpus() < 1:
        pytest.skip("needs a GPU")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={P}",
           "--master-addr", "127.0.0.1", "--master-port", str(29660 + P),
           os.path.join(ROOT, "tests", "mp_stress_worker.py"), "--iters", "300", "--layouts", "all"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT,
                       env=dict(os.environ, LANE_TEST_DEVICE="0"))
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "mp_stress_worker" in out and ": OK" in out, out[-4000:]


def _p8_env():
    return dict(os.environ, LANE_TEST_GPUS=str(1 if _ngpus() < 2 else 2))


def test_p8_ranks_sharing_gpus():
    """P = 8 through the multi-process path on a 1- or 2-GPU box (8 ranks on one
    GPU, or 4 + 4 with peers both local and over NVLink): every P = 8 layout
    (1x8, 2x4, 4x2, 8x1), simple / bulk stores / chunk claims / LL / LL128,
    fp32 / bf16 / int32, bit-exact vs the oracle. About 90 s on one B200
    (profiles/r02_p8_shared.txt)."""
    if _ngpus() < 1:
        pytest.skip("needs a GPU")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=8",
           "--master-addr", "127.0.0.1", "--master-port", "29671",
           os.path.join(ROOT, "tests", "mp_samedev_worker.py"), "--quick"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=_p8_env())
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "mp_samedev_worker: OK" in out, out[-4000:]


def test_p8_stress_sharing_gpus():
    """The exact stress at P = 8 (every layout, 300 calls each, up to 7 writers
    per destination) with the 8 ranks on one or two GPUs."""
    if _ngpus() < 1:
        pytest.skip("needs a GPU")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=8",
           "--master-addr", "127.0.0.1", "--master-port", "29672",
           os.path.join(ROOT, "tests", "mp_stress_worker.py"), "--iters", "300", "--layouts", "all"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=_p8_env())
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert out.count(": OK (0 bad calls") == 4, out[-4000:]


def test_p8_baseline_fullsize_sharing_gpus():
    """BASELINE configs[1] at P = 8 and full size (2x4, fp32, 1 GiB per rank)
    through the multi-process path with the 8 ranks on one or two GPUs: every
    output element of every rank bit-exact on the device
    (tools/p8_fullsize_check.py; profiles/r02_p8_fullsize_shared.txt)."""
    if _ngpus() < 1:
        pytest.skip("needs a GPU")
    import torch
    free = torch.cuda.mem_get_info(0)[0]
    if free < (48 << 30):
        pytest.skip("needs ~48 GiB free on GPU 0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=8",
           "--master-addr", "127.0.0.1", "--master-port", "29673",
           os.path.join(ROOT, "tools", "p8_fullsize_check.py"), "--layouts", "2x4", "--mib", "1024", "--calls", "1"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=_p8_env())
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "p8_fullsize_check 2x4 k=1 float32 1024 MiB/rank" in out and ": OK (2147483648 elements" in out, out[-4000:]
