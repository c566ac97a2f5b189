# round 2 (aw), 4 GPUs: the full GPU tier (every test, multi-GPU workers with graph
# replays, stress, watchdog) + smoke on the final code.
set -x
O=gpurun_out/r2aw; mkdir -p $O
timeout 2700 python -m pytest tests -m gpu -q > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "rc=$?" >> $O/smoke.txt
