# 1 GPU, as the driver's round end: pytest -m gpu, smoke, bench N=1, ncu launch list + full capture
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
( time timeout 1500 python -m pytest tests -x -q -m gpu ) > gpurun_out/e20_pytest_gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/e20_smoke.txt 2>&1
python bench.py > gpurun_out/e20_bench_n1.jsonl 2> gpurun_out/e20_bench_n1.err
python bench.py --steps 5 --warmup 3 > gpurun_out/e20_plain_launch.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/e20_launches_n1.csv \
    python bench.py --steps 5 --warmup 3 > gpurun_out/e20_ncu_launch.log 2>&1
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/e20_plain_full.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lane_tma -s 3 -c 1 -o gpurun_out/e20_prof_n1 \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/e20_ncu_full.log 2>&1
