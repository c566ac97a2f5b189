# 1 GPU: full gpu test suite (driver tier), smoke, N=1 bench
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
( time timeout 1500 python -m pytest tests -x -q -m gpu ) > gpurun_out/e29_pytest_gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/e29_smoke.txt 2>&1
python bench.py > gpurun_out/e29_bench_n1.jsonl 2> gpurun_out/e29_bench_n1.err
