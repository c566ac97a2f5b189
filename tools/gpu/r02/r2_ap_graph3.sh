# round 2 (ap), 4 GPUs: multi-GPU tier after the graph-case threshold fix.
set -x
O=gpurun_out/r2ap; mkdir -p $O
timeout 2400 python -m pytest tests/test_gpu_multigpu.py tests/test_gpu_emulated.py -m gpu -q -k "multigpu or stress or watchdog or graph" > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
