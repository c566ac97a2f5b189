# round 2 (x), 4 GPUs: chunk size / CTA budget at 128 MiB - 1 GiB, 3 layouts,
# 3 repeats (the r2w single-shot hints: 256 KiB chunks +3% at 1 GiB on 1x4).
set -x
O=gpurun_out/r2x; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
port=29960
for rep in 1 2 3; do
  for L in 1x4 4x1 2x2; do
    port=$((port+1))
    timeout 900 $TR --master-port $port tools/tune_mid.py --layout $L --mib 128 256 1024 --iters 20 --cfg "" \
      "LANE_CHUNK_BYTES=262144" "LANE_CHUNK_BYTES=524288" "LANE_CTAS_TOTAL=96" "LANE_CTAS_TOTAL=96,LANE_CHUNK_BYTES=262144" \
      | sed "s/^/$L /" >> $O/tune.txt 2>> $O/tune.err
  done
done
