# round 2 (g), 4 GPUs: where the 8-64 MiB band loses time. Steady-state traces
# (LL128 phase timeline; simple-protocol stall accounting) and a tuning grid of
# chunk geometry / CTA budgets at the mid sizes, 2x2 fp32 registered.
set -x
O=gpurun_out/r2g; mkdir -p $O
# parity of the new pull-push job set (LANE_DIRECT=4) on real peers first
timeout 600 python -m pytest tests/test_gpu_emulated.py -m gpu -x -q -k "parity_layouts and 4" > $O/pytest_mode4.txt 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29599 tests/mp_worker.py --quick > $O/mp_worker_quick.txt 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
for m in 8 16 32; do
  LANE_PROTO=ll128 timeout 300 $TR --master-port 2960$m tools/trace_run.py --layout 2x2 --mib $m --calls 20 > $O/trace_ll128_${m}.txt 2>&1
done
for m in 32 64; do
  LANE_PROTO=simple timeout 300 $TR --master-port 2961$m tools/trace_run.py --layout 2x2 --mib $m --calls 20 --register > $O/trace_simple_${m}.txt 2>&1
done
# simple protocol: chunk geometry at 24-96 MiB
timeout 900 $TR --master-port 29620 tools/tune_mid.py --layout 2x2 --mib 24 32 48 64 96 --iters 40 --nccl --cfg \
  "LANE_PROTO=simple" \
  "LANE_PROTO=simple,LANE_MIN_CHUNK_BYTES=65536" \
  "LANE_PROTO=simple,LANE_MIN_CHUNK_BYTES=65536,LANE_CHUNKS_PER_CTA=2" \
  "LANE_PROTO=simple,LANE_MIN_CHUNK_BYTES=65536,LANE_CHUNKS_PER_CTA=3" \
  "LANE_PROTO=simple,LANE_MIN_CHUNK_BYTES=32768,LANE_CHUNKS_PER_CTA=4" \
  "LANE_PROTO=simple,LANE_MIN_CHUNK_BYTES=32768,LANE_CHUNKS_PER_CTA=6" \
  "LANE_PROTO=simple,LANE_MIN_CHUNK_BYTES=65536,LANE_BULK_MIN_BYTES=1048576" \
  "LANE_PROTO=simple,LANE_MIN_CHUNK_BYTES=65536,LANE_STORE=lsu" \
  "LANE_PROTO=simple,LANE_DIRECT=3" \
  "LANE_PROTO=simple,LANE_DIRECT=4" \
  "LANE_PROTO=simple,LANE_DIRECT=4,LANE_MIN_CHUNK_BYTES=65536" \
  "LANE_PROTO=simple,LANE_DIRECT=4,LANE_MIN_CHUNK_BYTES=65536,LANE_CHUNKS_PER_CTA=2" \
  "LANE_PROTO=simple,LANE_CTAS_TOTAL=128" \
  "LANE_PROTO=simple,LANE_RELEASERS=2" \
  > $O/tune_simple.txt 2>&1
# LL128: CTA budget, U, sizes up to its 32 MiB capacity
timeout 900 $TR --master-port 29621 tools/tune_mid.py --layout 2x2 --mib 4 8 12 16 24 32 --iters 40 --cfg \
  "LANE_PROTO=ll128" \
  "LANE_PROTO=ll128,LANE_LL128_U1_MAX_BYTES=67108864" \
  "LANE_PROTO=ll128,LANE_LL_CTAS=128" \
  "LANE_PROTO=ll128,LANE_LL_CTAS=96" \
  "LANE_PROTO=ll128,LANE_LL_CTAS=74" \
  "LANE_PROTO=ll128,LANE_LL128_MIN_CHUNK_BYTES=65536" \
  > $O/tune_ll128.txt 2>&1
