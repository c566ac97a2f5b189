# 2 GPUs: busbw vs size at P=2 (1x2, 2x1) with NCCL ring, Alg.1 ring and approach 2 columns; P=2 bench line
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export BENCH_ARGS="--ring --approach2"
bash tools/sweep_sizes.sh 2 1x2 1024 gpurun_out/e22_sizes_p2.txt ""
bash tools/sweep_sizes.sh 2 2x1 1024 gpurun_out/e22_sizes_p2.txt ""
unset BENCH_ARGS
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29931 bench.py --gpus 2 > gpurun_out/e22_bench_n2.jsonl 2> gpurun_out/e22_bench_n2.err
