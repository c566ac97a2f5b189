#!/bin/bash
# BASELINE configs[4]: every layout NxG with N*G = P, k in {1,2,4,8}, int32 and fp32, 1 GiB per rank.
# usage: tools/scaling_matrix.sh P OUT.jsonl [extra bench args]
P=$1; OUT=$2; shift 2
port=29900
for N in 1 2 4 8; do
  [ $((P % N)) -ne 0 ] && continue
  G=$((P / N))
  for k in 1 2 4 8; do
    for dt in float32 int32; do
      port=$((port+1))
      nccl="--no-nccl"; [ $k -eq 1 ] && nccl=""
      timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$P --master-addr 127.0.0.1 \
        --master-port $port bench.py --gpus $P --layout ${N}x${G} --k $k --dtype $dt --no-e2e --steps 20 \
        --warmup 3 $nccl "$@" 2>/dev/null | grep '^{' >> $OUT
    done
  done
done
