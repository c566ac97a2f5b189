# 4 GPUs: chunk size / CTA count at mid sizes with bulk stores
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1"
for L in 2x2 4x1; do
$T --master-port 29961 tools/tune_mid.py --layout $L --mib 8 16 32 64 --iters 30 --cfg "LANE_PROTO=simple,LANE_STORE=bulk" \
  "LANE_PROTO=simple,LANE_STORE=bulk,LANE_MIN_CHUNK_BYTES=131072" "LANE_PROTO=simple,LANE_STORE=bulk,LANE_MIN_CHUNK_BYTES=262144" \
  "LANE_PROTO=simple,LANE_STORE=bulk,LANE_CTAS_TOTAL=74,LANE_MIN_CHUNK_BYTES=131072" \
  "LANE_PROTO=simple,LANE_STORE=bulk,LANE_MIN_CHUNK_BYTES=32768,LANE_CHUNKS_PER_CTA=2" \
  "LANE_PROTO=simple,LANE_STORE=bulk,LANE_RELEASERS=1" >> gpurun_out/e27_tune.txt 2>&1
done
