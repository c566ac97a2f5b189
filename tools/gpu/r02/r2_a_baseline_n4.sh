set -x
nvidia-smi -L
nvidia-smi nvlink -h > gpurun_out/r2a_nvlink_help.txt 2>&1
nvidia-smi nvlink -s -i 0 > gpurun_out/r2a_nvlink_status.txt 2>&1
nvidia-smi nvlink -gt d -i 0 > gpurun_out/r2a_nvlink_gt0.txt 2>&1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r2a_bench_n4.jsonl 2> gpurun_out/r2a_bench_n4.err
nvidia-smi nvlink -gt d -i 0 > gpurun_out/r2a_nvlink_gt0_after.txt 2>&1
nvidia-smi nvlink -gt r -i 0 > gpurun_out/r2a_nvlink_gtr_after.txt 2>&1
nvidia-smi topo -m > gpurun_out/r2a_topo.txt 2>&1
lscpu > gpurun_out/r2a_lscpu.txt; nproc >> gpurun_out/r2a_lscpu.txt
