# round 2 (p), 4 GPUs: LL128 with two warp steps in flight in D and E, A/B vs
# the previous build (tools/ab/liblane_head.so), 2x2 and 4x1, 2 repeats.
set -x
O=gpurun_out/r2p; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
port=29800
for rep in 1 2; do
  for L in 2x2 4x1; do
    port=$((port+1))
    timeout 600 $TR --master-port $port tools/tune_mid.py --layout $L --mib 1 2 4 8 16 24 32 --iters 50 \
      --cfg "LANE_PROTO=ll128" >> $O/ab_new_$L.txt 2>&1
    port=$((port+1))
    LANE_LIB_PATH=$PWD/tools/ab/liblane_head.so timeout 600 $TR --master-port $port tools/tune_mid.py --layout $L \
      --mib 1 2 4 8 16 24 32 --iters 50 --cfg "LANE_PROTO=ll128" >> $O/ab_old_$L.txt 2>&1
  done
done
