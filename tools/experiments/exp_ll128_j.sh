# Full GPU tier on 4 GPUs + smoke (current default build), then the LL128 warp-role split experiment (parity + P=4 sweeps)
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -4 > gpurun_out/j_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/j_pytest.txt 2>&1
cat gpurun_out/j_pytest.txt
cp paper_2508_13397_b200/liblane_allreduce.so /tmp/lib_def.so
cp build/var/lib_split.so paper_2508_13397_b200/liblane_allreduce.so
timeout 600 python -m pytest tests/test_gpu_emulated.py -x -q -k "ll128" 2>&1 | tail -2 > gpurun_out/j_split.txt
for L in 2x2 4x1; do BENCH_ARGS="--no-nccl" timeout 300 bash tools/sweep_sizes.sh 4 $L 64 gpurun_out/j_split.txt "LANE_PROTO=ll128"; done
cp /tmp/lib_def.so paper_2508_13397_b200/liblane_allreduce.so
cat gpurun_out/j_split.txt
