# round 2 (aa), 4 GPUs: dynamic chunk claims (LANE_DYN_CHUNKS=1) — parity
# (emulated job sets with 'd', repeated mixed-protocol calls, multi-GPU worker),
# then busbw static vs dynamic, P = 4 three layouts, 2 repeats.
set -x
O=gpurun_out/r2aa; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 1200 python -m pytest tests/test_gpu_emulated.py -m gpu -x -q -k "parity_layouts or whole_buffer or repeated_calls" > $O/pytest_emulated.txt 2>&1
port=30000
port=$((port+1)); timeout 900 $TR --master-port $port tests/mp_worker.py --quick > $O/mp_worker_quick.txt 2>&1
for rep in 1 2; do
  for L in 2x2 4x1 1x4; do
    port=$((port+1))
    timeout 900 $TR --master-port $port tools/tune_mid.py --layout $L --mib 32 48 64 128 256 1024 --iters 30 \
      --cfg "LANE_PROTO=simple" "LANE_PROTO=simple,LANE_DYN_CHUNKS=1" | sed "s/^/$L /" >> $O/ab.txt 2>> $O/ab.err
  done
done
port=$((port+1)); LANE_DYN_CHUNKS=1 LANE_PROTO=simple timeout 300 $TR --master-port $port tools/trace_run.py --layout 2x2 --mib 64 --calls 20 --register > $O/trace_dyn_64.txt 2>&1
port=$((port+1)); LANE_PROTO=simple timeout 300 $TR --master-port $port tools/trace_run.py --layout 2x2 --mib 64 --calls 20 --register > $O/trace_static_64.txt 2>&1
