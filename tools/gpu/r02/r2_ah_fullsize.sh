# round 2 (ah), 1 GPU: BASELINE-size parity with the whole-buffer device check.
set -x
O=gpurun_out/r2ah; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_emulated.py -m gpu -q -k "full_size" > $O/pytest_fullsize.txt 2>&1; echo "rc=$?" >> $O/pytest_fullsize.txt
