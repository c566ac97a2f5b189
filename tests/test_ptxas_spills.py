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
