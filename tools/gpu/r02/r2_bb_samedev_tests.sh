# round 2 (bb), 1 GPU: the ranks-sharing-one-GPU tests of tests/test_gpu_multigpu.py.
O=gpurun_out/r2bb; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_multigpu.py -m gpu -q -rs --durations=0 > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
