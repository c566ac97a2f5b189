# round 2 (ag), 1 GPU: ncu --set full of the LL128 kernel (line pairs) on the
# emulated 2x4 16 MiB/rank call, the same workload as the round-1/round-2 captures.
set -x
O=gpurun_out/r2ag; mkdir -p $O
LANE_PROTO=ll128 timeout 300 python tools/quick_time.py --layout 2x4 --mib 16 --iters 50 > $O/quick_ll128_16.txt 2>&1
LANE_PROTO=ll128 timeout 900 ncu --set full --clock-control none --import-source on -k regex:lane_ll128 -s 3 -c 1 \
  -o $O/prof_ll128_16mib python tools/quick_time.py --layout 2x4 --mib 16 --iters 1 > $O/ncu_ll128_16.log 2>&1
