# round 2 (bl), 1 GPU: the P = 8 full-size test with all 8 ranks on one GPU, as the 1-GPU tier runs it.
O=gpurun_out/r2bl; mkdir -p $O
timeout 100 python -m pytest tests/test_gpu_multigpu.py -m gpu -q -rs -k "p8_baseline" --durations=0 > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
