# full GPU test tier on 4 GPUs (multi-GPU parity incl. LL128, stress, watchdog), then default-protocol sweeps vs NCCL ring
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -15 > gpurun_out/d_pytest.txt
O=gpurun_out/d_sweep.txt
for L in 2x2 4x1 1x4; do timeout 400 bash tools/sweep_sizes.sh 4 $L 128 $O ""; done
for L in 1x2 2x1; do CUDA_VISIBLE_DEVICES=0,1 timeout 400 bash tools/sweep_sizes.sh 2 $L 128 $O ""; done
cat gpurun_out/d_pytest.txt $O
