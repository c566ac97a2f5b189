# LANE_PHASE2=ring on LL128: emulated parity (both protocols), multi-GPU parity (mp_worker ring2 / ring2_128), sweeps lane-ring2 P=4
timeout 900 python -m pytest tests/test_gpu_emulated.py -x -q -k "phase2 or ll128" 2>&1 | tail -3 > gpurun_out/k_pytest.txt
timeout 900 python -m pytest tests/test_gpu_multigpu.py -x -q -k "parity" 2>&1 | tail -3 >> gpurun_out/k_pytest.txt
cat gpurun_out/k_pytest.txt
O=gpurun_out/k_sweep.txt
for L in 2x2 4x1; do LANE_PHASE2=ring BENCH_ARGS="--no-nccl" timeout 400 bash tools/sweep_sizes.sh 4 $L 256 $O "" "LANE_PROTO=ll"; done
cat $O
