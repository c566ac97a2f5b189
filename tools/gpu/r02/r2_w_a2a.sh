# round 2 (w), 4 GPUs: the all-to-all layouts (1x4, 4x1) at 1 GiB — CTA budget
# and chunk size vs busbw; 2x2 for reference; plus the 4-GPU P2P microbenchmark.
set -x
O=gpurun_out/r2w; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
port=29940
for L in 1x4 4x1 2x2; do
  port=$((port+1))
  timeout 900 $TR --master-port $port tools/tune_mid.py --layout $L --mib 256 1024 --iters 20 --cfg "" \
    "LANE_CTAS_TOTAL=128" "LANE_CTAS_TOTAL=96" "LANE_CTAS_TOTAL=64" \
    "LANE_CHUNK_BYTES=262144" "LANE_CHUNK_BYTES=2097152" "LANE_RELEASERS=2" > $O/tune_$L.txt 2>&1
done
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/p2p_multi tools/p2p_multi.cu && timeout 600 tools/p2p_multi > $O/p2p_multi.txt 2>&1
