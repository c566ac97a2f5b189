# 4 GPUs: LL kernel with two granules per thread in flight: parity + LL sizes
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_emulated.py -x -q > gpurun_out/e21_pytest_emu.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multigpu.py -x -q > gpurun_out/e21_pytest_mp.txt 2>&1
T="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1"
for L in 2x2 4x1 1x4; do
$T --master-port 29921 tools/tune_mid.py --layout $L --mib 1 2 4 8 16 --iters 30 --nccl --cfg "LANE_PROTO=ll" >> gpurun_out/e21_tune.txt 2>&1
done
