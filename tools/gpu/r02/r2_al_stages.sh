# round 2 (al), 4 GPUs: TMA engine smem ring geometry (stages x KB: 4x48 default,
# 8x24, 6x32, 3x64) — simple protocol, 16 MiB - 1 GiB, 3 layouts, 2 repeats.
set -x
O=gpurun_out/r2al; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
port=30120
for rep in 1 2; do
  for lib in default s8x24 s6x32 s3x64; do
    if [ $lib = default ]; then unset LANE_LIB_PATH; else export LANE_LIB_PATH=$PWD/tools/ab/liblane_$lib.so; fi
    for L in 2x2 1x4 4x1; do
      port=$((port+1))
      timeout 600 $TR --master-port $port tools/tune_mid.py --layout $L --mib 16 32 64 128 1024 --iters 30 \
        --cfg "LANE_PROTO=simple" | sed "s/^/$lib $L /" >> $O/ab.txt 2>> $O/ab.err
    done
  done
done
