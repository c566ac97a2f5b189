# dev experiment (4 GPUs): several releaser warps: tuning + parity
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1"
$T --master-port 29841 tools/tune_mid.py --layout 2x2 --mib 4 8 16 32 64 256 1024 --iters 20 --cfg "" "LANE_RELEASERS=1" \
  "LANE_RELEASERS=2" "LANE_PROTO=simple" "LANE_PROTO=simple,LANE_RELEASERS=1" "LANE_PROTO=simple,LANE_MIN_CHUNK_BYTES=16384" \
  "LANE_PROTO=simple,LANE_CHUNKS_PER_CTA=8" "LANE_STORE=bulk" "LANE_STORE=lsu" > gpurun_out/e11_tune.txt 2>&1
for r in 1 4; do LANE_RELEASERS=$r timeout 120 python tools/quick_time.py --layout 2x4 --mib 1024 >> gpurun_out/e11_emu.txt 2>&1; done
timeout 900 python -m pytest tests/test_gpu_emulated.py -x -q > gpurun_out/e11_pytest_emu.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multigpu.py -x -q > gpurun_out/e11_pytest_mp.txt 2>&1
