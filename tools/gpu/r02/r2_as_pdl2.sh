# round 2 (as), 4 GPUs: PDL again now that the binding is no longer host-bound
# at small sizes — LANE_PDL=1 vs 0 by size, 2x2 and 1x4, 2 repeats.
set -x
O=gpurun_out/r2as; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
port=30600
for rep in 1 2; do
  for L in 2x2 1x4; do
    port=$((port+1))
    timeout 900 $TR --master-port $port tools/tune_mid.py --layout $L --mib 0.25 1 4 16 32 64 --iters 100 \
      --cfg "" "LANE_PDL=1" | sed "s/^/$L /" >> $O/ab.txt 2>> $O/ab.err
  done
done
