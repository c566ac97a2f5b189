# round 2 (ae), 1 GPU: the driver's 1-GPU tier on the final build (pytest -m gpu + smoke).
set -x
O=gpurun_out/r2ae; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q --durations=10 > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "rc=$?" >> $O/smoke.txt
