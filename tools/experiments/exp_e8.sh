# dev experiment (4 GPUs): fence-scope experiment + P=4 bench line
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1"
$T --master-port 29811 tools/tune_mid.py --layout 2x2 --mib 4 8 16 32 64 256 --cfg "" "LANE_FENCE_SCOPE_GPU=1" \
  "LANE_PROTO=simple" "LANE_PROTO=simple,LANE_FENCE_SCOPE_GPU=1" > gpurun_out/e8_tune.txt 2>&1
PYTHONUNBUFFERED=1 $T --master-port 29812 bench.py --gpus 4 > gpurun_out/e8_bench_n4.jsonl 2> gpurun_out/e8_bench_n4.err; echo "rc=$?" >> gpurun_out/e8_bench_n4.err
