# round 2 (z), 1 GPU: N = 1 bench + ncu launch list + full capture after the
# emulated chunk fix; the BASELINE configs[2] / configs[3] shapes emulated.
set -x
O=gpurun_out/r2z; mkdir -p $O
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench_n1.jsonl 2> $O/bench_n1.err
bash tools/gpu/lane_gpu.sh r2z ncu-n1
timeout 600 python bench.py --steps 20 --warmup 5 --layout 4x2 --k 4 --mib 256 --no-e2e > $O/bench_cfg2.jsonl 2> $O/bench_cfg2.err
timeout 600 python bench.py --steps 20 --warmup 5 --layout 8x1 --dtype bfloat16 --mib 512 --no-e2e > $O/bench_cfg3.jsonl 2> $O/bench_cfg3.err
timeout 600 python bench.py --steps 50 --warmup 5 --layout 2x4 --mib 1 --no-e2e --no-cpu > $O/bench_cfg1_1mib.jsonl 2> $O/bench_cfg1_1mib.err
