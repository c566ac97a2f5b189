# 4 GPUs: approach-2 parity (emulated + multi-GPU) and the standard / lane / approach-2 sweep
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_emulated.py -x -q -k "approach2 or ring or ll" > gpurun_out/e16_pytest_emu.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multigpu.py -x -q > gpurun_out/e16_pytest_mp.txt 2>&1
export BENCH_ARGS="--ring --approach2"
bash tools/sweep_sizes.sh 4 2x2 256 gpurun_out/e16_sizes.txt ""
