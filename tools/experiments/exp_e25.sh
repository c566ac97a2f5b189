# 4 GPUs: pull-all registered job set (LANE_DIRECT=3): parity + sizes vs push
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_emulated.py -x -q -k "parity_layouts or inplace" > gpurun_out/e25_pytest_emu.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multigpu.py -x -q > gpurun_out/e25_pytest_mp.txt 2>&1
T="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1"
for L in 2x2 4x1 1x4; do
$T --master-port 29951 tools/tune_mid.py --layout $L --mib 8 16 32 64 256 1024 --iters 20 --cfg "LANE_PROTO=simple" "LANE_PROTO=simple,LANE_DIRECT=3" "LANE_PROTO=simple,LANE_DIRECT=3,LANE_STORE=lsu" >> gpurun_out/e25_tune.txt 2>&1
done
