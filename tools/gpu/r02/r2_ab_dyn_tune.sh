# round 2 (ab), 4 GPUs: with dynamic claims, do smaller chunks pay now?
set -x
O=gpurun_out/r2ab; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
port=30020
for L in 2x2 4x1 1x4; do
  port=$((port+1))
  timeout 900 $TR --master-port $port tools/tune_mid.py --layout $L --mib 32 64 128 256 1024 --iters 30 --cfg \
    "LANE_PROTO=simple" "LANE_PROTO=simple,LANE_DYN_CHUNKS=1,LANE_MIN_CHUNK_BYTES=65536,LANE_CHUNKS_PER_CTA=8" \
    "LANE_PROTO=simple,LANE_DYN_CHUNKS=1,LANE_CHUNKS_PER_CTA=8" "LANE_PROTO=simple,LANE_DYN_CHUNKS=1,LANE_CHUNK_BYTES=262144" \
    | sed "s/^/$L /" >> $O/tune.txt 2>> $O/tune.err
done
