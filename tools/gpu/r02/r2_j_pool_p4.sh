# round 2 (j), 4 GPUs: LL128 with the pooled tail (LANE_LL128_STATIC_PCT),
# parity first (emulated LL128 cases, multi-GPU quick worker, stress), then
# busbw vs the static share, and LL128 vs simple around the threshold.
set -x
O=gpurun_out/r2j; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_emulated.py -m gpu -x -q -k "ll128" > $O/pytest_ll128.txt 2>&1
timeout 600 $TR --master-port 29670 tests/mp_worker.py --quick > $O/mp_worker_quick.txt 2>&1
timeout 600 $TR --master-port 29671 tests/mp_stress_worker.py --iters 500 --layouts all > $O/stress.txt 2>&1
for L in 2x2 4x1 1x4; do
  timeout 900 $TR --master-port 2968${L:0:1} tools/tune_mid.py --layout $L --mib 2 4 8 16 24 32 48 --iters 50 --cfg \
    "LANE_PROTO=ll128,LANE_LL128_STATIC_PCT=100" "LANE_PROTO=ll128,LANE_LL128_STATIC_PCT=75" \
    "LANE_PROTO=ll128,LANE_LL128_STATIC_PCT=50" "LANE_PROTO=ll128,LANE_LL128_STATIC_PCT=25" \
    "LANE_PROTO=ll128,LANE_LL128_STATIC_PCT=0" "LANE_PROTO=simple" > $O/tune_$L.txt 2>&1
done
i=0
for pct in 100 50 0; do
  i=$((i+1))
  LANE_LL128_STATIC_PCT=$pct LANE_PROTO=ll128 timeout 300 $TR --master-port 2969$i tools/trace_run.py --layout 2x2 --mib 32 --calls 20 > $O/trace_ll128_32_s$pct.txt 2>&1
done
