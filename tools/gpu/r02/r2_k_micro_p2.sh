# round 2 (k), 2 GPUs: LL128 line-push microbenchmark (store flavour x U x CTAs,
# bidirectional), parity of the LL128 kernel after the phase restructure.
set -x
O=gpurun_out/r2k; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ll128_micro tools/ll128_micro.cu && timeout 600 tools/ll128_micro > $O/ll128_micro.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_emulated.py -m gpu -x -q -k "ll128" > $O/pytest_ll128.txt 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29700 tests/mp_worker.py --quick > $O/mp_worker_quick.txt 2>&1
