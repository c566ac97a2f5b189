# round 2 (n), 1 GPU: back-to-back kernel gap vs parameter size and PDL.
set -x
O=gpurun_out/r2n; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/launch_micro tools/launch_micro.cu && timeout 300 tools/launch_micro > $O/launch_micro.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > $O/bench_n1.jsonl 2> $O/bench_n1.err
