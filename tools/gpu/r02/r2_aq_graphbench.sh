# round 2 (aq), 4 GPUs: eager calls vs the same calls replayed from a CUDA graph.
set -x
O=gpurun_out/r2aq; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for L in 2x2 1x4; do
  timeout 900 $TR --master-port 3040${L:0:1} tools/graph_bench.py --layout $L --mib 0.25 1 4 16 64 > $O/graph_$L.txt 2>&1
done
