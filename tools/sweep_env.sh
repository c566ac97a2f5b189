#!/bin/bash
# Run the multi-GPU bench under several LANE_* settings (dev tool).
# usage: tools/sweep_env.sh NGPU OUT "ENV1" "ENV2" ... ; extra bench args in $BENCH_ARGS
NG=$1; OUT=$2; shift 2
port=29600
for cfg in "$@"; do
  port=$((port+1))
  echo "### $cfg $BENCH_ARGS" >> $OUT
  env $cfg timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$NG --master-addr 127.0.0.1 \
     --master-port $port bench.py --gpus $NG --no-e2e --no-cpu --steps 20 --warmup 3 $BENCH_ARGS 2>&1 | grep '^{' \
     | python -c "import json,sys; [print(json.dumps({k: d.get(k) for k in ('value','ms_per_step','verified')} | {'layout': d['config']['layout'], 'k': d['config']['procs_per_gpu'], 'plan': d['config']['plan'], 'nccl': (d.get('nccl_ring') or {}).get('value')})) for d in map(json.loads, sys.stdin)]" >> $OUT 2>&1
done
