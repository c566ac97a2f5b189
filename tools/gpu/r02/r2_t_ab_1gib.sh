# round 2 (t), 4 GPUs: 1 GiB A/B on one box — the build at the start of this
# session (tools/ab/liblane_r2start.so), the PDL build before the deferred
# handshake (tools/ab/liblane_fcc.so) and the current build, layouts 1x4 / 4x1 /
# 2x2, 3 alternating repeats; then the copy-engine microbenchmark (2 GPUs).
set -x
O=gpurun_out/r2t; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
port=29880
for rep in 1 2 3; do
  for lib in r2start fcc cur; do
    if [ $lib = cur ]; then unset LANE_LIB_PATH; else export LANE_LIB_PATH=$PWD/tools/ab/liblane_$lib.so; fi
    for L in 1x4 4x1 2x2; do
      port=$((port+1))
      timeout 600 $TR --master-port $port tools/tune_mid.py --layout $L --mib 256 1024 --iters 20 --cfg "" \
        | sed "s/^/$lib $L /" >> $O/ab_1gib.txt 2>> $O/ab_1gib.err
    done
  done
done
unset LANE_LIB_PATH
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ce_micro tools/ce_micro.cu && timeout 300 tools/ce_micro > $O/ce_micro.txt 2>&1
