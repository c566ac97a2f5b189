# LL128 with dynamic (per-phase atomic) line claiming: GPU parity (emulated + multi-GPU + stress), forced-LL128 sweeps at P=4/P=2, trace 32 MiB
timeout 900 python -m pytest tests/test_gpu_emulated.py -x -q -k "ll128 or mixed or ring" 2>&1 | tail -3 > gpurun_out/i_pytest.txt
timeout 900 python -m pytest tests/test_gpu_multigpu.py -x -q 2>&1 | tail -3 >> gpurun_out/i_pytest.txt
cat gpurun_out/i_pytest.txt
O=gpurun_out/i_sweep.txt
for L in 2x2 4x1 1x4; do BENCH_ARGS="--no-nccl" timeout 300 bash tools/sweep_sizes.sh 4 $L 64 $O "LANE_PROTO=ll128"; done
for L in 1x2 2x1; do CUDA_VISIBLE_DEVICES=0,1 BENCH_ARGS="--no-nccl" timeout 300 bash tools/sweep_sizes.sh 2 $L 64 $O "LANE_PROTO=ll128"; done
LANE_PROTO=ll128 timeout 120 python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29650 tools/trace_run.py --layout 2x2 --mib 32 --calls 20 > gpurun_out/i_trace.txt 2>&1
cat $O
