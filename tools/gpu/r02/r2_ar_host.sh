# round 2 (ar), 2 GPUs: host-side cost per allreduce call (binding vs bare C ABI vs a torch launch).
set -x
O=gpurun_out/r2ar; mkdir -p $O
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 30501 tools/host_overhead.py > $O/host.txt 2>&1
