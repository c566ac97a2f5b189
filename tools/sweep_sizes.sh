#!/bin/bash
# busbw vs size for several LANE_* settings (dev tool). usage: tools/sweep_sizes.sh NGPU LAYOUT MAXMIB OUT "ENV"...
NG=$1; L=$2; MX=$3; OUT=$4; shift 4
port=29800
for cfg in "$@"; do
  port=$((port+1))
  env $cfg timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$NG --master-addr 127.0.0.1 \
     --master-port $port bench.py --gpus $NG --layout $L --mib $MX --sweep /tmp/sw_$port.jsonl > /dev/null 2>&1
  python - "$cfg" /tmp/sw_$port.jsonl >> $OUT <<'PY'
import json, sys
rows = [json.loads(l) for l in open(sys.argv[2])]
print(sys.argv[1], rows[0]["layout"] if rows else "?", " ".join(f"{r['bytes']>>20}M:{r['busbw']:.0f}/{r['nccl_ring_busbw']:.0f}{'' if r['verified'] else '!'}" for r in rows))
PY
done
