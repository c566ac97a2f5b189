# 4 GPUs: parity, P=4 bench line, busbw-vs-size sweeps (2x2, 4x1, 1x4) with NCCL ring and our Alg.1 ring
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/e13_smoke.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_emulated.py -x -q > gpurun_out/e13_pytest_emu.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multigpu.py -x -q > gpurun_out/e13_pytest_mp.txt 2>&1
T="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1"
$T --master-port 29861 bench.py --gpus 4 > gpurun_out/e13_bench_n4.jsonl 2> gpurun_out/e13_bench_n4.err; echo "rc=$?" >> gpurun_out/e13_bench_n4.err
export BENCH_ARGS="--ring"
bash tools/sweep_sizes.sh 4 2x2 1024 gpurun_out/e13_sizes.txt ""
bash tools/sweep_sizes.sh 4 4x1 1024 gpurun_out/e13_sizes.txt ""
bash tools/sweep_sizes.sh 4 1x4 1024 gpurun_out/e13_sizes.txt ""
