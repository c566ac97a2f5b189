# LL128 protocol: GPU parity (emulated), then per-protocol busbw sweeps at P=4 (3 layouts) and P=2 (2 layouts)
timeout 600 python -m pytest tests/test_gpu_emulated.py -x -q -k "ll128 or mixed or ll_cta" 2>&1 | tail -5 > gpurun_out/c_pytest.txt
O=gpurun_out/c_sweep.txt
for L in 2x2 4x1 1x4; do
  BENCH_ARGS="--no-nccl" timeout 300 bash tools/sweep_sizes.sh 4 $L 64 $O "LANE_PROTO=ll128" "LANE_PROTO=ll"
  BENCH_ARGS="--no-nccl" timeout 300 bash tools/sweep_sizes.sh 4 $L 64 $O "LANE_PROTO=simple"
done
for L in 1x2 2x1; do
  CUDA_VISIBLE_DEVICES=0,1 BENCH_ARGS="--no-nccl" timeout 300 bash tools/sweep_sizes.sh 2 $L 64 $O "LANE_PROTO=ll128" "LANE_PROTO=ll" "LANE_PROTO=simple"
done
cat gpurun_out/c_pytest.txt $O
