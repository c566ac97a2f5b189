# 4 GPUs: no end-of-call barrier (F5 flags + zero-byte E waits): parity + sweeps
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_emulated.py -x -q > gpurun_out/e18_pytest_emu.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multigpu.py -x -q > gpurun_out/e18_pytest_mp.txt 2>&1
T="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1"
for L in 2x2 4x1 1x4; do
$T --master-port 29901 tools/tune_mid.py --layout $L --mib 4 8 16 32 64 256 1024 --iters 20 --cfg "" "LANE_PROTO=simple" >> gpurun_out/e18_tune.txt 2>&1
done
timeout 120 python tools/quick_time.py --layout 2x4 --mib 1024 >> gpurun_out/e18_tune.txt 2>&1
