set -x
nvidia-smi -L
timeout 600 python -m pytest tests/test_gpu_emulated.py -x -q -k "ll128 or mixed" 2>&1 | tail -15 > gpurun_out/g1_pytest.txt
cat gpurun_out/g1_pytest.txt
BENCH_ARGS="--no-nccl" timeout 400 bash tools/sweep_sizes.sh 4 2x2 128 gpurun_out/g1_sweep.txt "LANE_PROTO=ll128" "LANE_PROTO=ll" 
timeout 300 bash tools/sweep_sizes.sh 4 2x2 128 gpurun_out/g1_sweep.txt "" 
cat gpurun_out/g1_sweep.txt
