# round 2 (bf), 1 GPU: the P = 8 ranks-sharing-GPUs tests as the driver's 1-GPU tier runs them.
O=gpurun_out/r2bf; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_multigpu.py -m gpu -q -rs --durations=0 -k "p8 or sharing" > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
