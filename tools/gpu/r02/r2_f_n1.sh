# round 2 (f), 1 GPU: driver tier (pytest -m gpu + smoke), N=1 bench line, ncu
# launch list + --set full capture of the dominant kernel (lane_tma_kernel, 2x4
# fp32 1 GiB/rank) on the build without local memory, and an ncu capture of the
# LL128 kernel (emulated 2x4, 16 MiB/rank).
set -x
O=gpurun_out/r2f; mkdir -p $O
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
bash tools/gpu/lane_gpu.sh r2f tests
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench_n1.jsonl 2> $O/bench_n1.err
bash tools/gpu/lane_gpu.sh r2f ncu-n1
LANE_PROTO=ll128 timeout 300 python tools/quick_time.py --layout 2x4 --mib 16 --iters 50 > $O/quick_ll128_16.txt 2>&1
LANE_PROTO=ll128 timeout 900 ncu --set full --clock-control none --import-source on -k regex:lane_ll128 -s 3 -c 1 \
  -o $O/prof_ll128_16mib python tools/quick_time.py --layout 2x4 --mib 16 --iters 1 > $O/ncu_ll128_16.log 2>&1
