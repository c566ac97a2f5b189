# round 2 (m), 4 GPUs: deferred start handshake (scratch-only jobs run while
# it completes) + layout-dependent protocol ranges. Full GPU test tier first
# (multi-GPU parity, mismatch/timeout tests), then A/B vs the previous build
# (tools/ab/liblane_fcc.so) on the simple protocol, then the P = 4 sweep.
set -x
O=gpurun_out/r2m; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
for rep in 1 2; do
  LANE_PROTO=simple timeout 900 $TR --nproc-per-node 4 --master-port 2972$rep tools/tune_mid.py --layout 2x2 \
    --mib 16 32 64 128 --iters 50 --cfg "" >> $O/ab_new.txt 2>&1
  LANE_LIB_PATH=$PWD/tools/ab/liblane_fcc.so LANE_PROTO=simple timeout 900 $TR --nproc-per-node 4 --master-port 2973$rep \
    tools/tune_mid.py --layout 2x2 --mib 16 32 64 128 --iters 50 --cfg "" >> $O/ab_old.txt 2>&1
done
LANE_PROTO=simple timeout 300 $TR --nproc-per-node 4 --master-port 29741 tools/trace_run.py --layout 2x2 --mib 64 --calls 20 --register > $O/trace_simple_64.txt 2>&1
for L in 2x2 4x1 1x4; do
  timeout 900 $TR --nproc-per-node 4 --master-port 2975${L:0:1} bench.py --gpus 4 --layout $L --sweep $O/sweep_p4.jsonl --mib 256 > $O/sweep_p4_$L.log 2>&1
done
