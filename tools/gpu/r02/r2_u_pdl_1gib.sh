# round 2 (u), 4 GPUs: is PDL the 1 GiB 1x4 / 4x1 loss? current build with
# LANE_PDL=1 / 0 and the session-start build, 3 alternating repeats.
set -x
O=gpurun_out/r2u; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
port=29900
for rep in 1 2 3; do
  for cfg in pdl1 pdl0 r2start; do
    if [ $cfg = r2start ]; then export LANE_LIB_PATH=$PWD/tools/ab/liblane_r2start.so; else unset LANE_LIB_PATH; fi
    if [ $cfg = pdl0 ]; then export LANE_PDL=0; else unset LANE_PDL; fi
    for L in 1x4 4x1; do
      port=$((port+1))
      timeout 600 $TR --master-port $port tools/tune_mid.py --layout $L --mib 64 1024 --iters 20 --cfg "" \
        | sed "s/^/$cfg $L /" >> $O/ab.txt 2>> $O/ab.err
    done
  done
done
