# round 2 (af), 4 GPUs: producer scan order — earliest ready phase first
# (default) vs latest first (LANE_PRIO_LATE=1), simple protocol, 2 repeats.
set -x
O=gpurun_out/r2af; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
port=30060
for rep in 1 2; do
  for L in 2x2 4x1 1x4; do
    port=$((port+1))
    timeout 900 $TR --master-port $port tools/tune_mid.py --layout $L --mib 16 32 64 128 256 1024 --iters 30 \
      --cfg "LANE_PROTO=simple" "LANE_PROTO=simple,LANE_PRIO_LATE=1" | sed "s/^/$L /" >> $O/ab.txt 2>> $O/ab.err
  done
done
