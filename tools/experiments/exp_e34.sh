# 4 GPUs: long stress runs (every layout) + the multi-GPU pytest file
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T="timeout 900 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for L in 2x2 4x1 1x4; do
  $T --nproc-per-node=4 --master-port 29991 tests/mp_stress_worker.py --iters 5000 --layout $L >> gpurun_out/e34_stress.txt 2>&1
done
$T --nproc-per-node=2 --master-port 29992 tests/mp_stress_worker.py --iters 5000 --layout 1x2 >> gpurun_out/e34_stress.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_multigpu.py -x -q > gpurun_out/e34_pytest_mp.txt 2>&1
