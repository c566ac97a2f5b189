# round 2 (ad), 1 GPU: the driver's 1-GPU tier on the final build (pytest -m gpu
# + smoke) — includes the multi-round few-CTA chunk-claims test.
set -x
O=gpurun_out/r2ad; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -x -q --durations=15 > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "rc=$?" >> $O/smoke.txt
