# 4 GPUs: bf16 sweep (4x1, the shape of BASELINE configs[3] at P=4) and int32 sweep (2x2)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
BENCH_ARGS="--dtype bfloat16" bash tools/sweep_sizes.sh 4 4x1 512 gpurun_out/e31_sizes.txt "LANE_TAG=bf16"
BENCH_ARGS="--dtype int32" bash tools/sweep_sizes.sh 4 2x2 1024 gpurun_out/e31_sizes.txt "LANE_TAG=int32"
