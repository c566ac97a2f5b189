# round 2 (d): clock-backed evidence at P = 4 and P = 2:
# busbw vs size per layout (3 repeats, whole-buffer verification, NCCL ring /
# x4 PPG / default beside), the configs[4] matrix, the NCCL algorithm probe, and
# the stress test on all layouts with fp32/bf16 bit-exact checks.
set -x
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
OUT=gpurun_out/r2d
mkdir -p $OUT
for L in 2x2 4x1 1x4; do
  timeout 900 $TR --nproc-per-node 4 --master-port 29561 bench.py --gpus 4 --layout $L --sweep $OUT/sweep_p4.jsonl --mib 1024 > $OUT/sweep_p4_$L.log 2>&1
done
for L in 1x2 2x1; do
  timeout 900 $TR --nproc-per-node 2 --master-port 29562 bench.py --gpus 2 --layout $L --sweep $OUT/sweep_p2.jsonl --mib 1024 > $OUT/sweep_p2_$L.log 2>&1
done
timeout 900 $TR --nproc-per-node 4 --master-port 29563 tools/matrix.py --out $OUT/matrix_p4.jsonl --dtypes float32 int32 bfloat16 > $OUT/matrix_p4.log 2>&1
timeout 900 $TR --nproc-per-node 2 --master-port 29564 tools/matrix.py --out $OUT/matrix_p2.jsonl --dtypes float32 int32 > $OUT/matrix_p2.log 2>&1
NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,NVLS,TUNING NCCL_DEBUG_FILE=$OUT/nccl_probe_p4.%h.%p.log timeout 600 $TR --nproc-per-node 4 --master-port 29565 tools/nccl_algo_probe.py > $OUT/nccl_probe_p4.jsonl 2> $OUT/nccl_probe_p4.err
timeout 1200 $TR --nproc-per-node 4 --master-port 29566 tests/mp_stress_worker.py --iters 1500 --layouts all > $OUT/stress_p4.txt 2>&1
