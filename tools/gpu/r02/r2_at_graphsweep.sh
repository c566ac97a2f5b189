# round 2 (at), 4 GPUs: eager vs CUDA-graph replay, busbw vs size 1 MiB - 1 GiB,
# every P = 4 and P = 2 layout, whole-buffer verified after the last replay, clocks.
set -x
O=gpurun_out/r2at; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
port=30700
for L in 2x2 4x1 1x4; do
  port=$((port+1)); timeout 1200 $TR --nproc-per-node 4 --master-port $port tools/graph_bench.py --layout $L \
    --mib 1 2 4 8 16 32 64 128 256 512 1024 --out $O/graph_p4.jsonl > $O/graph_p4_$L.log 2>&1
done
for L in 1x2 2x1; do
  port=$((port+1)); timeout 1200 $TR --nproc-per-node 2 --master-port $port tools/graph_bench.py --layout $L \
    --mib 1 2 4 8 16 32 64 128 256 512 1024 --out $O/graph_p2.jsonl > $O/graph_p2_$L.log 2>&1
done
