# 4 GPUs: 2x2 mid sizes with the 128 KiB chunk: store mode, chunks per CTA, bulk threshold
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1"
$T --master-port 29981 tools/tune_mid.py --layout 2x2 --mib 8 16 32 64 --iters 30 --cfg "LANE_PROTO=simple" \
  "LANE_PROTO=simple,LANE_STORE=lsu" "LANE_PROTO=simple,LANE_STORE=bulk" "LANE_PROTO=simple,LANE_CHUNKS_PER_CTA=2" \
  "LANE_PROTO=simple,LANE_CHUNKS_PER_CTA=8" "LANE_PROTO=simple,LANE_MIN_CHUNK_BYTES=196608" \
  "LANE_PROTO=simple,LANE_STORE=bulk,LANE_CHUNKS_PER_CTA=2,LANE_MIN_CHUNK_BYTES=65536" > gpurun_out/e30_tune.txt 2>&1
