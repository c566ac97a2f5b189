# 1 GPU: compute-sanitizer memcheck over small emulated runs of every kernel
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 120 python tools/sanitize_small.py > gpurun_out/e33_plain.txt 2>&1 && \
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_small.py > gpurun_out/e33_memcheck.txt 2>&1
echo "rc=$?" >> gpurun_out/e33_memcheck.txt
