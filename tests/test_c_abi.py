"""The boundary is plain C: tests/c_abi_example.c (C99) compiles with
``gcc -std=c99 -Wall -Wextra -pedantic -Werror`` against include/lane_allreduce.h,
links with liblane_allreduce.so and runs the host-only entry points on CPU."""
import os
import shutil
import subprocess

import pytest

from paper_2508_13397_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("gcc") is None, reason="needs gcc")
def test_c99_client_builds_and_runs(tmp_path):
    _lib.load()  # the library exists (raises otherwise)
    libdir = os.path.dirname(_lib.LIB_PATH)
    exe = tmp_path / "c_abi_example"
    cc = ["gcc", "-std=c99", "-Wall", "-Wextra", "-pedantic", "-Werror", "-I", os.path.join(ROOT, "include"),
          os.path.join(ROOT, "tests", "c_abi_example.c"), "-L", libdir, "-llane_allreduce",
          f"-Wl,-rpath,{libdir}", "-o", str(exe)]
    r = subprocess.run(cc, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stdout + r.stderr
    out = r.stdout
    assert "topology rank 5: node 1 gpu 1 group 4 5 6 7 lane 1 5" in out
    assert "partition units 16 first {round 0 l 0 c 0 g 0 a 0 start 0 end 64}" in out
    assert "init_rank(nodes=0) -> -1 comm NULL" in out and "nodes" in out
