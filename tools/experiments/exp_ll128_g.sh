# Ring (Alg. 1) on LL128: emulated ring parity (LL and LL128), multi-GPU parity at P=4 (mp_worker incl. ring on LL128),
# then standard (ring) vs lane sweeps at P=4 2x2 and P=2 1x2
timeout 900 python -m pytest tests/test_gpu_emulated.py -x -q -k "ring" 2>&1 | tail -4 > gpurun_out/g_pytest.txt
timeout 900 python -m pytest tests/test_gpu_multigpu.py -x -q -k "parity" 2>&1 | tail -4 >> gpurun_out/g_pytest.txt
O=gpurun_out/g_sweep.txt
BENCH_ARGS="--ring --no-nccl" timeout 400 bash tools/sweep_sizes.sh 4 2x2 1024 $O ""
CUDA_VISIBLE_DEVICES=0,1 BENCH_ARGS="--ring --no-nccl" timeout 400 bash tools/sweep_sizes.sh 2 1x2 1024 $O ""
cat gpurun_out/g_pytest.txt $O
