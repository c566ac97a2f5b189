"""Summarise an ncu report (--set full) of the lane kernel into a small JSON
that is committed under profiles/ and read by bench.py for roofline.traffic.

python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r01_ncu_n1_summary.json \
    --workload "2x4 emulated fp32 1024 MiB/rank" --bytes-per-rank 1073741824 --ranks 8
"""
import argparse
import csv
import io
import json
import subprocess

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "dram__bytes.sum.per_second": "dram_rate",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum": "tma_load_bytes",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__shared_mem_per_block_dynamic": "smem_dynamic",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9, "us": 1e-6,
         "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1, "second": 1,
         "byte/s": 1, "Kbyte/s": 1e3, "Mbyte/s": 1e6, "Gbyte/s": 1e9, "Tbyte/s": 1e12}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("out")
    ap.add_argument("--workload", required=True)
    ap.add_argument("--bytes-per-rank", type=int, required=True)
    ap.add_argument("--ranks", type=int, required=True)
    a = ap.parse_args()
    txt = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        k = {"kernel": d.get("Kernel Name")}
        for key, name in KEYS.items():
            if key in d and d[key] not in ("", None):
                try:
                    v = float(d[key].replace(",", ""))
                except ValueError:
                    continue
                k[name] = v * SCALE.get(u.get(key, ""), 1) if u.get(key) in SCALE else v
        if "dram_read" in k and "dram_write" in k:
            k["dram_bytes"] = k["dram_read"] + k["dram_write"]
            k["dram_bytes_per_rank_per_byte"] = k["dram_bytes"] / (a.ranks * a.bytes_per_rank)
        kernels.append(k)
    out = {"report": a.report, "workload": a.workload, "bytes_per_rank": a.bytes_per_rank, "ranks": a.ranks,
           "kernels": kernels}
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
