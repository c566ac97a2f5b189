# 2 GPUs: watchdog test
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 250 python -m pytest tests/test_gpu_multigpu.py -x -q -k watchdog > gpurun_out/e26_watchdog.txt 2>&1; echo "rc=$?" >> gpurun_out/e26_watchdog.txt
nvidia-smi --query-gpu=index,utilization.gpu,memory.used --format=csv >> gpurun_out/e26_watchdog.txt
