# round 2 (ao), 4 GPUs: CUDA-graph support — full GPU tier (emulated graph test,
# multi-GPU workers with graph replays, stress) after the test fix.
set -x
O=gpurun_out/r2ao; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "rc=$?" >> $O/smoke.txt
