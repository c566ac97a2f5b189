# round 2 (e), 1 GPU: N=1 bench line, ncu launch list + --set full capture of the
# dominant kernel (lane_tma_kernel, 2x4 fp32 1 GiB/rank), and an ncu capture of the
# LL128 kernel (emulated 2x4, 16 MiB/rank) after the local-memory removal.
set -x
O=gpurun_out/r2e; mkdir -p $O
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench_n1.jsonl 2> $O/bench_n1.err
bash tools/gpu/lane_gpu.sh r2e ncu-n1
for pr in ll128; do
  LANE_PROTO=$pr timeout 300 python tools/quick_time.py --layout 2x4 --mib 16 --iters 50 > $O/quick_${pr}_16.txt 2>&1
  LANE_PROTO=$pr timeout 900 ncu --set full --clock-control none --import-source on -k regex:lane_ll128 -s 3 -c 1 \
    -o $O/prof_${pr}_16mib python tools/quick_time.py --layout 2x4 --mib 16 --iters 1 > $O/ncu_${pr}_16.log 2>&1
done
LANE_PROTO=ll timeout 300 python tools/quick_time.py --layout 2x4 --mib 1 --iters 50 > $O/quick_ll_1.txt 2>&1
