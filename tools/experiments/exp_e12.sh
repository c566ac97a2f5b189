# dev experiment (4 GPUs): LL16 parity + tuning
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/e12_smoke.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_emulated.py -x -q > gpurun_out/e12_pytest_emu.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multigpu.py -x -q > gpurun_out/e12_pytest_mp.txt 2>&1
T="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1"
$T --master-port 29851 tools/tune_mid.py --layout 2x2 --mib 1 2 4 8 16 32 64 --iters 30 --nccl --cfg "" \
  "LANE_LL_PACKET=32" "LANE_PROTO=ll" "LANE_PROTO=ll,LANE_LL_PACKET=32" "LANE_PROTO=simple" > gpurun_out/e12_tune.txt 2>&1
$T --master-port 29852 tools/tune_mid.py --layout 4x1 --mib 1 4 8 16 32 --iters 30 --cfg "" "LANE_PROTO=ll" "LANE_PROTO=simple" > gpurun_out/e12_tune_4x1.txt 2>&1
$T --master-port 29853 tools/tune_mid.py --layout 1x4 --mib 1 4 8 16 32 --iters 30 --cfg "" "LANE_PROTO=ll" "LANE_PROTO=simple" > gpurun_out/e12_tune_1x4.txt 2>&1
