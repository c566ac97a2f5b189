#!/bin/bash
# busbw vs size for several LANE_* settings (dev tool).
# usage: tools/sweep_sizes.sh NGPU LAYOUT MAXMIB OUT "ENV"...   (extra bench args in $BENCH_ARGS)
# prints per size: ours/NCCL-ring[/our Alg.1 ring] and the protocol (l = LL, L = LL128, s = simple)
NG=$1; L=$2; MX=$3; OUT=$4; shift 4
port=29800
for cfg in "$@"; do
  port=$((port+1))
  rm -f /tmp/sw_$port.jsonl
  env $cfg timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$NG --master-addr 127.0.0.1 \
     --master-port $port bench.py --gpus $NG --layout $L --mib $MX --sweep /tmp/sw_$port.jsonl $BENCH_ARGS > /dev/null 2>&1
  python - "$cfg" /tmp/sw_$port.jsonl $L >> $OUT <<'PY'
import json, os, sys
rows = [json.loads(l) for l in open(sys.argv[2])] if os.path.exists(sys.argv[2]) else []
def cell(r):
    s = f"{r['bytes']>>20}M:{r['busbw']:.0f}/{r['nccl_ring_busbw']:.0f}"
    if "lane_ring_alg1_busbw" in r:
        s += f"/{r['lane_ring_alg1_busbw']:.0f}"
    if "approach2_busbw" in r:
        s += f"/a{r['approach2_busbw']:.0f}"
    return s + {"ll128": "L"}.get(r.get("protocol"), r.get("protocol", "?")[0]) + ("" if r["verified"] else "!")
print(sys.argv[1] or "default", sys.argv[3], " ".join(cell(r) for r in rows) if rows else "NO OUTPUT")
PY
done
