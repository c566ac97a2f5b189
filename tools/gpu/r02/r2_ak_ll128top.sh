# round 2 (ak), 1 GPU: LL128 at the top of its default range on P = 8 layouts (emulated).
set -x
O=gpurun_out/r2ak; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_emulated.py -m gpu -q -k "ll128_default_range_top or graph_capture" > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
