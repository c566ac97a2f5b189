"""DESIGN.md §8's tables are the renders of committed, clock-backed profiles
(tools/design_tables.py): every table row the tool renders from each file
named here appears verbatim in DESIGN.md, and every rendered file reports 0
rows without a clean clock record."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = [
    ["profiles/r02_sweep_p4_final.jsonl"],
    ["profiles/r02_sweep_p2_final.jsonl"],
    ["profiles/r02_sweep_bf16_p4.jsonl"],
    ["--matrix", "profiles/r02_matrix_p4_final.jsonl"],
    ["--matrix", "profiles/r02_matrix_p2_final.jsonl"],
    ["--std", "profiles/r02_sweep_p4_final.jsonl"],
    ["--std", "profiles/r02_sweep_p2_std.jsonl"],
]


@pytest.mark.parametrize("args", CASES, ids=lambda a: " ".join(a))
def test_design_table_rendered_from_profile(args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "design_tables.py"), *args],
                       capture_output=True, text=True, cwd=ROOT, timeout=120)
    assert r.returncode == 0, r.stderr
    assert "0 rows without a clean clock record" in r.stdout
    rows = [ln for ln in r.stdout.splitlines() if ln.startswith("| ")]
    assert rows
    with open(os.path.join(ROOT, "DESIGN.md")) as f:
        design = f.read()
    missing = [ln for ln in rows if ln not in design]
    assert not missing, missing[:3]
