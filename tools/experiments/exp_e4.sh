# dev experiment (4 GPUs): full parity + LL phase traces + default sweep
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_emulated.py -x -q > gpurun_out/e4_pytest_emu.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multigpu.py -x -q > gpurun_out/e4_pytest_mp.txt 2>&1
port=29750
for L in 2x2 4x1; do for M in 1 4; do
 port=$((port+1))
 echo "### $L $M MiB" >> gpurun_out/e4_trace.txt
 timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port $port tools/trace_run.py --layout $L --mib $M 2>/dev/null | grep -v "^\*\|OMP" >> gpurun_out/e4_trace.txt
done; done
timeout 120 python tools/trace_run.py --emulated --layout 2x2 --mib 1 >> gpurun_out/e4_trace.txt 2>&1
export BENCH_ARGS="--ring"
bash tools/sweep_sizes.sh 4 2x2 1024 gpurun_out/e4_sizes.txt ""
