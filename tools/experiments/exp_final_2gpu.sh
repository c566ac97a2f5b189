# 2 GPUs: full pytest -m gpu (1-GPU tier + P=2 multi-GPU parity, stress, watchdog) and smoke on the final build
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -4 > gpurun_out/n_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1 >> gpurun_out/n_pytest.txt
cat gpurun_out/n_pytest.txt
