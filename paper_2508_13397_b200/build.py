"""Build the in-tree shared libraries with nvcc for sm_100a.

  paper_2508_13397_b200/liblane_allreduce.so   product: kernels + C ABI
  seeded_inputs/libseeded_fill.so              test/bench input generator

Usage: python -m paper_2508_13397_b200.build [--force]
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2",
                 "-shared", "--expt-relaxed-constexpr"]

TARGETS = [
    {
        "out": os.path.join(PKG, "liblane_allreduce.so"),
        "srcs": [os.path.join(PKG, "csrc", "lane_host.cu")],
        "deps": [os.path.join(PKG, "csrc", f) for f in sorted(os.listdir(os.path.join(PKG, "csrc")))
                 if f.endswith((".h", ".cuh"))] + [os.path.join(ROOT, "include", "lane_allreduce.h")],
        "log": os.path.join(PKG, "csrc", "ptxas_lane_allreduce.log"),
    },
    {
        "out": os.path.join(ROOT, "seeded_inputs", "libseeded_fill.so"),
        "srcs": [os.path.join(ROOT, "seeded_inputs", "csrc", "seeded_fill.cu")],
        "deps": [],
        "log": None,
    },
]


def _stale(t) -> bool:
    if not os.path.exists(t["out"]):
        return True
    mt = os.path.getmtime(t["out"])
    return any(os.path.getmtime(f) > mt for f in t["srcs"] + t["deps"] + [__file__])


def build(force: bool = False, verbose: bool = False) -> list[str]:
    built = []
    for t in TARGETS:
        if not force and not _stale(t):
            continue
        extra = os.environ.get("LANE_NVCC_FLAGS", "").split()  # dev experiments (e.g. -DLANE_TMA_STAGE_KB=24)
        cmd = [NVCC] + COMMON + extra + (["-Xptxas", "-v"] if t["log"] else []) + t["srcs"] + ["-o", t["out"]]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if t["log"]:
            with open(t["log"], "w") as f:
                f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed for {t['out']}")
        if verbose:
            print("built", t["out"])
        built.append(t["out"])
    return built


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
