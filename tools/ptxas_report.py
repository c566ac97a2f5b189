"""Per-function stack frame / spill bytes / registers from the ptxas -v log of
the library build (paper_2508_13397_b200/csrc/ptxas_lane_allreduce.log) and the
STL/LDL instruction counts from `cuobjdump -sass` of the built .so.

    python tools/ptxas_report.py [--sass]
"""
import re
import subprocess
import sys
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LOG = os.path.join(ROOT, "paper_2508_13397_b200", "csrc", "ptxas_lane_allreduce.log")
SO = os.path.join(ROOT, "paper_2508_13397_b200", "liblane_allreduce.so")


def ptxas_table():
    rows, cur = {}, None
    for line in open(LOG):
        m = re.search(r"Function properties for (\S+)", line)
        if m:
            cur = m.group(1)
            continue
        m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m and cur:
            rows.setdefault(cur, {}).update(stack=int(m.group(1)), spill_st=int(m.group(2)), spill_ld=int(m.group(3)))
            continue
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m:
            cur = m.group(1)
            continue
        m = re.search(r"Used (\d+) registers", line)
        if m and cur:
            rows.setdefault(cur, {})["regs"] = int(m.group(1))
    return rows


def sass_local_counts():
    out = subprocess.run(["cuobjdump", "-sass", SO], capture_output=True, text=True).stdout
    cnt, cur = {}, None
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            cnt[cur] = [0, 0]
            continue
        if cur and re.search(r"\bSTL", line):
            cnt[cur][0] += 1
        if cur and re.search(r"\bLDL", line):
            cnt[cur][1] += 1
    return cnt


if __name__ == "__main__":
    rows = ptxas_table()
    sass = sass_local_counts() if "--sass" in sys.argv else {}
    print(f"{'function':70s} regs stack spill_st spill_ld" + ("  STL  LDL" if sass else ""))
    for f, r in rows.items():
        if not f.startswith("_ZN4lane") or "kernel" not in f:
            continue
        s = f"{f[:70]:70s} {r.get('regs', '-'):>4} {r.get('stack', 0):>5} {r.get('spill_st', 0):>8} {r.get('spill_ld', 0):>8}"
        if sass:
            c = sass.get(f, [0, 0])
            s += f" {c[0]:>4} {c[1]:>4}"
        print(s)
