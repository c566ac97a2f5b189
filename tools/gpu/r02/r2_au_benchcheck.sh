# round 2 (au), 2 GPUs: bench.py sanity on the final build (N = 1 default, N = 2 self-launch).
set -x
O=gpurun_out/r2au; mkdir -p $O
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_n1.jsonl 2> $O/bench_n1.err
timeout 900 python bench.py --gpus 2 --steps 20 --warmup 5 > $O/bench_n2.jsonl 2> $O/bench_n2.err
