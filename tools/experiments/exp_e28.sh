# 4 GPUs: parity, final P=4 sweeps (2x2, 4x1, 1x4) and bench line
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_emulated.py -x -q > gpurun_out/e28_pytest_emu.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multigpu.py -x -q > gpurun_out/e28_pytest_mp.txt 2>&1
T="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1"
$T --master-port 29971 bench.py --gpus 4 > gpurun_out/e28_bench_n4.jsonl 2> gpurun_out/e28_bench_n4.err
export BENCH_ARGS="--ring --approach2"
bash tools/sweep_sizes.sh 4 2x2 1024 gpurun_out/e28_sizes.txt ""
bash tools/sweep_sizes.sh 4 4x1 1024 gpurun_out/e28_sizes.txt ""
bash tools/sweep_sizes.sh 4 1x4 1024 gpurun_out/e28_sizes.txt ""
