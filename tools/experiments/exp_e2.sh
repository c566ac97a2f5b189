# dev experiment: parity (emulated + P=2) and busbw vs size per protocol
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_emulated.py -x -q > gpurun_out/e2_pytest_emu.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_multigpu.py -x -q > gpurun_out/e2_pytest_mp.txt 2>&1
bash tools/sweep_sizes.sh 2 1x2 256 gpurun_out/e2_sizes.txt "LANE_PROTO=simple" "LANE_PROTO=simple LANE_STORE=bulk" "LANE_PROTO=ll" "LANE_PROTO=ll LANE_LL_CTAS=64"
bash tools/sweep_sizes.sh 2 2x1 64 gpurun_out/e2_sizes.txt "LANE_PROTO=simple" "LANE_PROTO=ll"
