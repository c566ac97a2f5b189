# LL128 protocol: emulated parity, then P=4 2x2 busbw sweeps for U = 2 (default), 4, 1 lines per group per warp step
set -x
timeout 600 python -m pytest tests/test_gpu_emulated.py -x -q -k "ll128 or mixed or ll_cta" 2>&1 | tail -5 > gpurun_out/b_pytest.txt
cat gpurun_out/b_pytest.txt
O=gpurun_out/b_sweep.txt
BENCH_ARGS="--no-nccl" timeout 300 bash tools/sweep_sizes.sh 4 2x2 64 $O "LANE_PROTO=ll128"
cp paper_2508_13397_b200/liblane_allreduce.so /tmp/lib_u2.so
for U in 4 1; do
  cp build/var/lib_u$U.so paper_2508_13397_b200/liblane_allreduce.so
  echo "U=$U" >> $O
  BENCH_ARGS="--no-nccl" timeout 300 bash tools/sweep_sizes.sh 4 2x2 64 $O "LANE_PROTO=ll128"
done
cp /tmp/lib_u2.so paper_2508_13397_b200/liblane_allreduce.so
LANE_PROTO=ll128 timeout 120 python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29650 tools/trace_run.py --layout 2x2 --mib 16 --calls 20 > gpurun_out/b_trace.txt 2>&1
cat $O
