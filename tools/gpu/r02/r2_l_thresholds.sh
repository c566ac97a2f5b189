# round 2 (l), 4 GPUs: protocol crossover points per layout — LL vs LL128
# below 2 MiB, LL128 vs simple at 16-64 MiB (LL128 capacity raised to 64 MiB
# for the measurement); P = 4 (three layouts) and P = 2 (two layouts).
set -x
O=gpurun_out/r2l; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
port=29710
for P in 4 2; do
  if [ $P = 4 ]; then LS="2x2 4x1 1x4"; else LS="1x2 2x1"; fi
  for L in $LS; do
    port=$((port+1))
    timeout 900 $TR --nproc-per-node $P --master-port $port tools/tune_mid.py --layout $L \
      --mib 0.25 0.5 1 2 4 --iters 100 --cfg "LANE_PROTO=ll" "LANE_PROTO=ll128" > $O/small_p${P}_$L.txt 2>&1
    port=$((port+1))
    timeout 900 $TR --nproc-per-node $P --master-port $port tools/tune_mid.py --layout $L \
      --mib 12 16 24 32 48 64 --iters 40 --cfg "LANE_PROTO=ll128,LANE_LL128_MAX_BYTES=67108864" "LANE_PROTO=simple" \
      > $O/mid_p${P}_$L.txt 2>&1
  done
done
