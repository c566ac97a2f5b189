cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm --format=csv > gpurun_out/e1_smi.txt
port=29700
for L in 1x2 2x1; do for M in 8 64; do for ST in lsu bulk; do
 port=$((port+1))
 echo "### $L $M MiB LANE_STORE=$ST" >> gpurun_out/e1_trace.txt
 LANE_STORE=$ST timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port $port tools/trace_run.py --layout $L --mib $M >> gpurun_out/e1_trace.txt 2>&1
done; done; done
bash tools/sweep_sizes.sh 2 1x2 256 gpurun_out/e1_sizes.txt "LANE_STORE=lsu" "LANE_STORE=bulk" "LANE_CTAS_TOTAL=32" "LANE_CTAS_TOTAL=32 LANE_STORE=bulk" "LANE_CTAS_TOTAL=16 LANE_CHUNKS_PER_CTA=2"
