"""bench.py helpers the measurement contract rests on (CPU): the busbw
formula (nccl-tests' bus bandwidth, 2(P-1)/P of the message per unit time),
the clock record parsed from the nvidia-smi fallback (throttle reasons are
what makes a run rejected), the sweep sizes and the N = 1 roofline bytes."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_busbw_closed_forms():
    S, ms = 1 << 30, 2.0
    assert bench.busbw(S, 1, ms) == S / 2e-3 / 1e9
    assert abs(bench.busbw(S, 2, ms) - S / 2e-3 / 1e9) < 1e-9          # 2(P-1)/P = 1
    assert abs(bench.busbw(S, 4, ms) - 1.5 * S / 2e-3 / 1e9) < 1e-9
    assert abs(bench.busbw(S, 8, ms) - 1.75 * S / 2e-3 / 1e9) < 1e-9


def test_method_hbm_bytes():
    S = 1 << 30
    assert bench.method_hbm_bytes(8, 1, S) == 2 * S                     # no phase 1 / 3: read + write
    assert bench.method_hbm_bytes(2, 4, S) == int(S * 3.25)
    assert bench.method_hbm_bytes(4, 2, S) == int(S * 3.5)


def test_clock_record_from_nvidia_smi_csv(tmp_path):
    c = bench.Clocks([0, 1])
    c.out = str(tmp_path / "clk.csv")
    with open(c.out, "w") as f:
        f.write("0, 1965, 1965, 700.1, Not Active, Not Active, Not Active, Not Active\n")
        f.write("1, 1950, 1965, 690.0, Not Active, Not Active, Not Active, Active\n")
        f.write("0, 1965, 1965, 701.0, Not Active, Not Active, Not Active, Not Active\n")
        f.write("garbage line\n")
    s = c.summary()
    assert s["samples"] == 3 and s["sm_mhz"] == 1965 and s["sm_max_mhz"] == 1965 and s["sm_min_mhz"] == 1950
    assert s["reasons"] == ["sw_power_cap"]
    with open(c.out, "a") as f:
        f.write("1, 1400, 1965, 500.0, Active, Not Active, Not Active, Not Active\n")
    assert "hw_slowdown" in c.summary()["reasons"]


def test_clock_record_empty():
    c = bench.Clocks([0])
    c.out = "/nonexistent/clk.csv"
    s = c.summary()
    assert s["samples"] == 0 and s["sm_mhz"] is None


def test_sweep_sizes():
    class A:
        sizes = None
        mib = 1024.0
    assert bench.sweep_sizes(A) == [float(2 ** i) for i in range(11)]
    A.sizes = "1,16,64"
    assert bench.sweep_sizes(A) == [1.0, 16.0, 64.0]
