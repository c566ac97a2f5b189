# LL128 U=1 below 4 MiB: emulated parity, multi-GPU parity, default sweeps P=4 (3 layouts) and P=2 up to 32 MiB
timeout 900 python -m pytest tests/test_gpu_emulated.py -x -q -k "ll128 or mixed" 2>&1 | tail -2 > gpurun_out/m_pytest.txt
timeout 900 python -m pytest tests/test_gpu_multigpu.py -x -q -k "parity or stress" 2>&1 | tail -2 >> gpurun_out/m_pytest.txt
cat gpurun_out/m_pytest.txt
O=gpurun_out/m_sweep.txt
for L in 2x2 4x1 1x4; do timeout 300 bash tools/sweep_sizes.sh 4 $L 32 $O ""; done
for L in 1x2 2x1; do CUDA_VISIBLE_DEVICES=0,1 timeout 300 bash tools/sweep_sizes.sh 2 $L 32 $O ""; done
cat $O
