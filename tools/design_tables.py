"""Render DESIGN.md §8's measurement tables from the committed, clock-backed
profiles (sweep / matrix JSONL written by bench.py --sweep and
tools/matrix.py), so every number in §8 is read from a file whose rows carry
an NVML clock record — nothing typed by hand.

python tools/design_tables.py profiles/r02_sweep_p4.jsonl profiles/r02_sweep_p2.jsonl \
    --matrix profiles/r02_matrix_p4.jsonl profiles/r02_matrix_p2.jsonl
"""
import argparse
import json
from collections import OrderedDict

LETTER = {"ll": "l", "ll128": "L", "simple": ""}


def rows(path):
    with open(path) as f:
        return [json.loads(x) for x in f if x.strip()]


def clocks_ok(r):
    c = r.get("clocks") or {}
    return bool(c.get("samples")) and not (set(c.get("reasons", [])) &
                                           {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"})


def sweep_table(paths):
    out = []
    for path in paths:
        rs = [r for r in rows(path) if r.get("verified")]
        bad = [r for r in rs if not clocks_ok(r)]
        by = OrderedDict()
        for r in rs:
            by.setdefault(r["layout"], []).append(r)
        sizes = sorted({r["bytes"] >> 20 for r in rs})
        P = None
        out.append(f"`{path}` (median of {rs[0].get('repeats', 1)} repeats; ours / NCCL ring; "
                   f"l = LL, L = LL128, plain = simple; {len(bad)} rows without a clean clock record)\n")
        out.append("| layout | " + " | ".join(f"{m} MiB" for m in sizes) + " |")
        out.append("|---" * (len(sizes) + 1) + "|")
        for lay, rr in by.items():
            cells = {r["bytes"] >> 20: r for r in rr}
            line = [lay]
            for m in sizes:
                r = cells.get(m)
                if r is None:
                    line.append("—")
                    continue
                ring = r.get("nccl_ring_busbw")
                win = ring is None or r["busbw"] >= ring
                v = f"{r['busbw']:.0f}{LETTER.get(r['protocol'], '')}"
                line.append((f"**{v}**" if win else v) + (f" / {ring:.0f}" if ring is not None else ""))
            out.append("| " + " | ".join(line) + " |")
        out.append("")
    return "\n".join(out)


def std_table(paths):
    """The paper's standard-vs-lane comparison (fig:std_vs_lane, P L401, L457)
    from sweep rows that carry the Alg. 1 ring and approach 2 columns."""
    out = []
    for path in paths:
        rs = [r for r in rows(path) if r.get("verified") and "lane_ring_alg1_busbw" in r]
        bad = [r for r in rs if not clocks_ok(r)]
        out.append(f"`{path}` (busbw GB/s, median of {rs[0].get('repeats', 1)}; lane and approach 2 whole-buffer "
                   f"verified bit-exactly, ring on its first 2^16 elements within the per-hop bound; {len(bad)} rows without a clean clock record)\n")
        out.append("| layout | MiB per rank | lane method | Alg. 1 ring (ours) | lane / ring | approach 2 | NCCL ring |")
        out.append("|---|---|---|---|---|---|---|")
        for r in rs:
            out.append(f"| {r['layout']} | {r['bytes'] >> 20} | {r['busbw']:.0f}{LETTER.get(r['protocol'], '')} | "
                       f"{r['lane_ring_alg1_busbw']:.0f}{LETTER.get(r.get('ring_protocol'), '')} | "
                       f"{r['busbw'] / r['lane_ring_alg1_busbw']:.2f}× | "
                       f"{r['approach2_busbw']:.0f} | {r.get('nccl_ring_busbw', float('nan')):.0f} |"
                       if "approach2_busbw" in r else
                       f"| {r['layout']} | {r['bytes'] >> 20} | {r['busbw']:.0f} | {r['lane_ring_alg1_busbw']:.0f} | "
                       f"{r['busbw'] / r['lane_ring_alg1_busbw']:.2f}× | — | {r.get('nccl_ring_busbw', float('nan')):.0f} |")
        out.append("")
    return "\n".join(out)


def matrix_table(paths):
    out = []
    for path in paths:
        rs = rows(path)
        lane = [r for r in rs if r.get("impl") == "lane" and r.get("verified")]
        P = lane[0]["P"]
        ks = sorted({r["k"] for r in lane})
        dts = [d for d in ("float32", "int32", "bfloat16") if any(r["dtype"] == d for r in lane)]
        ring = {r["dtype"]: r["busbw"] for r in rs if r.get("impl") == "nccl_ring"}
        ppg = {r["dtype"]: r["busbw"] for r in rs if r.get("impl") == "nccl_ring_x4ppg"}
        out.append(f"`{path}` (P = {P}, 1 GiB per rank, busbw GB/s, median of 3; every lane cell whole-buffer "
                   f"verified; {sum(not clocks_ok(r) for r in rs)} rows without a clean clock record)\n")
        out.append("| layout | dtype | " + " | ".join(f"k={k}" for k in ks) + " | NCCL ring | NCCL ×4 PPG |")
        out.append("|---" * (len(ks) + 4) + "|")
        for lay in sorted({r["layout"] for r in lane}):
            for d in dts:
                cell = {r["k"]: r["busbw"] for r in lane if r["layout"] == lay and r["dtype"] == d}
                out.append(f"| {lay} | {d} | " + " | ".join(f"{cell[k]:.0f}" if k in cell else "—" for k in ks) +
                           f" | {ring.get(d, float('nan')):.0f} | {ppg.get(d, float('nan')):.0f} |")
        out.append("")
    return "\n".join(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("sweeps", nargs="*")
    ap.add_argument("--matrix", nargs="*", default=[])
    ap.add_argument("--std", nargs="*", default=[], help="sweeps with --ring --approach2 columns")
    a = ap.parse_args()
    if a.sweeps:
        print(sweep_table(a.sweeps))
    if a.matrix:
        print(matrix_table(a.matrix))
    if a.std:
        print(std_table(a.std))


if __name__ == "__main__":
    main()
