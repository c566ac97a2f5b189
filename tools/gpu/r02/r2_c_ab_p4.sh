# round 2 (c): A/B of the round-1 library build (tools/ab/liblane_r01.so) vs the
# current build on the same 4-GPU box, 2x2 fp32 registered, several sizes.
set -x
run() {  # $1 = lib label, $2 = MiB
  if [ "$1" = r01 ]; then export LANE_LIB_PATH=$PWD/tools/ab/liblane_r01.so; else unset LANE_LIB_PATH; fi
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29544 \
    bench.py --gpus 4 --steps 30 --warmup 5 --mib $2 --no-e2e --no-cpu --no-nccl --no-staged \
    | sed "s/^/$1 $2 /" >> gpurun_out/r2c_ab.txt 2>> gpurun_out/r2c_ab.err
}
for rep in 1 2 3; do
  for mib in 1024 64 32 16; do
    run r01 $mib
    run new $mib
  done
done
