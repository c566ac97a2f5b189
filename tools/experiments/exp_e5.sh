# dev experiment (4 GPUs): parity + mid-size tuning of the simple protocol
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_emulated.py -x -q > gpurun_out/e5_pytest_emu.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multigpu.py -x -q > gpurun_out/e5_pytest_mp.txt 2>&1
T="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1"
$T --master-port 29911 tools/tune_mid.py --layout 2x2 --mib 4 8 16 32 64 --nccl --cfg "" "LANE_PROTO=simple" \
  "LANE_PROTO=simple,LANE_CTAS_TOTAL=74" "LANE_PROTO=simple,LANE_CTAS_TOTAL=37" \
  "LANE_PROTO=simple,LANE_CHUNKS_PER_CTA=1" "LANE_PROTO=simple,LANE_CHUNKS_PER_CTA=2" \
  "LANE_PROTO=simple,LANE_MIN_CHUNK_BYTES=65536" "LANE_PROTO=simple,LANE_STORE=bulk" \
  "LANE_PROTO=simple,LANE_CTAS_TOTAL=74,LANE_CHUNKS_PER_CTA=2" > gpurun_out/e5_tune_2x2.txt 2>&1
$T --master-port 29912 tools/tune_mid.py --layout 4x1 --mib 4 8 16 32 64 --nccl --cfg "" "LANE_PROTO=simple" \
  "LANE_PROTO=simple,LANE_CTAS_TOTAL=74" "LANE_PROTO=simple,LANE_CHUNKS_PER_CTA=1" > gpurun_out/e5_tune_4x1.txt 2>&1
