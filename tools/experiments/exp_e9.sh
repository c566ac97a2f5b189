# dev experiment (4 GPUs): release master parity + mid-size tuning
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_emulated.py -x -q > gpurun_out/e9_pytest_emu.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multigpu.py -x -q > gpurun_out/e9_pytest_mp.txt 2>&1
T="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1"
$T --master-port 29821 tools/tune_mid.py --layout 2x2 --mib 4 8 16 32 64 256 1024 --iters 20 --cfg "" "LANE_REL_MASTER=0" \
  "LANE_PROTO=simple" "LANE_PROTO=simple,LANE_STORE=bulk" "LANE_STORE=lsu" "LANE_PROTO=simple,LANE_MIN_CHUNK_BYTES=16384" \
  "LANE_PROTO=simple,LANE_CHUNKS_PER_CTA=8" > gpurun_out/e9_tune.txt 2>&1
$T --master-port 29822 tools/tune_mid.py --layout 4x1 --mib 4 8 16 32 64 256 --iters 20 --cfg "" "LANE_PROTO=simple" > gpurun_out/e9_tune_4x1.txt 2>&1
$T --master-port 29823 tools/tune_mid.py --layout 1x4 --mib 4 8 16 32 64 256 --iters 20 --cfg "" "LANE_PROTO=simple" > gpurun_out/e9_tune_1x4.txt 2>&1
for st in lsu bulk; do LANE_STORE=$st timeout 120 python tools/quick_time.py --layout 2x4 --mib 1024 >> gpurun_out/e9_emu.txt 2>&1; done
