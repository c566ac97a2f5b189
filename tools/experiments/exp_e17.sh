# 2 GPUs: release-fence microbenchmark + steady-state trace of the registered path at mid sizes
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fence_micro tools/fence_micro.cu && timeout 300 tools/fence_micro > gpurun_out/e17_fence.txt 2>&1
T="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1"
port=29890
for M in 16 64; do
 port=$((port+1))
 echo "### 1x2 $M MiB registered steady state" >> gpurun_out/e17_trace.txt
 $T --master-port $port tools/trace_run.py --layout 1x2 --mib $M --calls 20 --register 2>/dev/null | grep -v "^\*\|OMP" >> gpurun_out/e17_trace.txt
done
