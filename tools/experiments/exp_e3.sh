# dev experiment (4 GPUs): parity incl. LL + ring, busbw vs size per protocol / store mode
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_emulated.py -x -q -k "ring or ll or mixed" > gpurun_out/e3_pytest_emu.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multigpu.py -x -q > gpurun_out/e3_pytest_mp.txt 2>&1
export BENCH_ARGS="--ring"
bash tools/sweep_sizes.sh 4 2x2 1024 gpurun_out/e3_sizes.txt "" "LANE_STORE=lsu" "LANE_LL_THRESHOLD_BYTES=16777216"
bash tools/sweep_sizes.sh 4 4x1 256 gpurun_out/e3_sizes.txt ""
bash tools/sweep_sizes.sh 4 1x4 256 gpurun_out/e3_sizes.txt ""
for st in lsu bulk; do LANE_STORE=$st timeout 120 python tools/quick_time.py --layout 2x4 --mib 1024 >> gpurun_out/e3_emu.txt 2>&1; done
