"""Verdict r1 #4 as a regression guard: no kernel of the library has a stack
frame or spills (ptxas -v log written by the build, tools/ptxas_report.py),
except the non-default lane-ring LL instantiations (`LANE_PHASE2=ring`,
lane_ll_kernel<DT, true>), whose few bytes DESIGN §6 records."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))

import ptxas_report  # noqa: E402

ALLOWED = ("_ZN4lane2ll14lane_ll_kernelILi0ELb1EEEvNS_10LaneParamsE",
           "_ZN4lane2ll14lane_ll_kernelILi1ELb1EEEvNS_10LaneParamsE",
           "_ZN4lane2ll14lane_ll_kernelILi2ELb1EEEvNS_10LaneParamsE")


def test_kernels_have_no_local_memory():
    rows = ptxas_report.ptxas_table()
    kernels = {k: v for k, v in rows.items() if "kernel" in k}
    assert len(kernels) >= 20, sorted(kernels)
    bad = {k: v for k, v in kernels.items()
           if k not in ALLOWED and (v.get("stack", 0) or v.get("spill_st", 0) or v.get("spill_ld", 0))}
    assert not bad, bad
    for k in ALLOWED:
        if k in kernels:
            assert kernels[k].get("spill_st", 0) <= 16, (k, kernels[k])


def test_sass_no_local_memory_and_bulk_copies():
    """SASS of the built library (cuobjdump, no GPU needed): no STL/LDL in any
    kernel but the allowed lane-ring LL instantiations, and the TMA engine
    kernels issue bulk copies (UBLKCP) and mbarrier operations (SYNCS)."""
    import re
    import shutil
    import subprocess
    import pytest
    if not os.path.exists(ptxas_report.SO) or shutil.which("cuobjdump") is None:
        pytest.skip("library not built or cuobjdump missing")
    out = subprocess.run(["cuobjdump", "-sass", ptxas_report.SO], capture_output=True, text=True,
                         timeout=300).stdout
    funcs, cur = {}, None
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = {"local": 0, "ublkcp": 0, "syncs": 0}
            continue
        if cur is None:
            continue
        if re.search(r"\b(STL|LDL)\b", line):
            funcs[cur]["local"] += 1
        if "UBLKCP" in line:
            funcs[cur]["ublkcp"] += 1
        if "SYNCS." in line:
            funcs[cur]["syncs"] += 1
    kernels = {k: v for k, v in funcs.items() if k.startswith("_ZN4lane") and "kernel" in k}
    assert len(kernels) >= 20
    bad = {k: v["local"] for k, v in kernels.items() if k not in ALLOWED and v["local"]}
    assert not bad, bad
    tma = {k: v for k, v in kernels.items() if "lane_tma_kernel" in k}
    assert tma and all(v["ublkcp"] > 0 and v["syncs"] > 0 for v in tma.values()), tma
