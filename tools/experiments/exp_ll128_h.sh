# LL128 variants at P=4 2x2 (sizes 1-64 MiB, LANE_PROTO=ll128): default (U=2, 512 thr), U=1, U=4, 256 threads (2 CTAs/SM),
# 256 threads U=4, weak stores; then a steady-state phase trace at 32 MiB
O=gpurun_out/h_sweep.txt
cp paper_2508_13397_b200/liblane_allreduce.so /tmp/lib_def.so
BENCH_ARGS="--no-nccl" timeout 300 bash tools/sweep_sizes.sh 4 2x2 64 $O "LANE_PROTO=ll128"
for v in u1 u4 t256 t256u4 weak; do
  cp build/var/lib_$v.so paper_2508_13397_b200/liblane_allreduce.so
  echo "variant $v" >> $O
  BENCH_ARGS="--no-nccl" timeout 300 bash tools/sweep_sizes.sh 4 2x2 64 $O "LANE_PROTO=ll128"
done
cp /tmp/lib_def.so paper_2508_13397_b200/liblane_allreduce.so
LANE_PROTO=ll128 timeout 120 python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29650 tools/trace_run.py --layout 2x2 --mib 32 --calls 20 > gpurun_out/h_trace.txt 2>&1
cat $O
