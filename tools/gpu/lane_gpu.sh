#!/bin/bash
# lane_gpu.sh — the one driver for GPU measurements of this repo (run on a
# gpurun box from the repo root; every output goes under gpurun_out/<tag>/).
#
#   bash tools/gpu/lane_gpu.sh TAG tests               # pytest -m gpu + smoke()
#   bash tools/gpu/lane_gpu.sh TAG bench N [args]      # bench.py line at N GPUs (N=1: emulated)
#   bash tools/gpu/lane_gpu.sh TAG sweep P LAYOUT MAXMIB [bench args]
#                                                      # busbw vs size, 3 repeats, clocks, NCCL ring/x4 PPG/default
#   bash tools/gpu/lane_gpu.sh TAG protocols P LAYOUT MAXMIB
#                                                      # the sweep once per LANE_PROTO (ll, ll128, simple)
#   bash tools/gpu/lane_gpu.sh TAG matrix P [matrix args]   # BASELINE configs[4]: layouts x k x dtypes at 1 GiB
#   bash tools/gpu/lane_gpu.sh TAG stress P ITERS      # every layout, int32/fp32/bf16 bit-exact back-to-back calls
#   bash tools/gpu/lane_gpu.sh TAG ncu-n1 [bench args] # ncu launch list (time per launch) + one --set full capture
#                                                      #   of the dominant kernel, N = 1 bench command
#   bash tools/gpu/lane_gpu.sh TAG nccl-probe P        # NCCL's algorithm choice with NCCL_ALGO unset (NVLS?)
#
# Environment settings (LANE_*) pass through, e.g. LANE_PROTO=simple bash ... .
# Round-1 experiments ran as one-off scripts (tools/experiments/README.md lists
# what each measured); their commands are subsumed by these subcommands.
set -u
TAG=$1; CMD=$2; shift 2
OUT=gpurun_out/$TAG
mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
port() { echo $((29700 + RANDOM % 200)); }
case $CMD in
  tests)
    timeout 1800 python -m pytest tests -m gpu -x -q > $OUT/pytest.txt 2>&1; echo "rc=$?" >> $OUT/pytest.txt
    timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; echo "rc=$?" >> $OUT/smoke.txt ;;
  bench)
    N=$1; shift
    timeout 1200 python bench.py --gpus $N "$@" > $OUT/bench_n$N.jsonl 2> $OUT/bench_n$N.err ;;
  sweep)
    P=$1; L=$2; M=$3; shift 3
    timeout 1200 $TR --nproc-per-node $P --master-port $(port) bench.py --gpus $P --layout $L --mib $M \
      --sweep $OUT/sweep_p$P.jsonl "$@" > $OUT/sweep_p${P}_$L.log 2>&1 ;;
  protocols)
    P=$1; L=$2; M=$3; shift 3
    for pr in ll ll128 simple; do
      LANE_PROTO=$pr timeout 1200 $TR --nproc-per-node $P --master-port $(port) bench.py --gpus $P --layout $L \
        --mib $M --no-nccl --sweep $OUT/protocols_p${P}_$pr.jsonl "$@" > $OUT/protocols_p${P}_${L}_$pr.log 2>&1
    done ;;
  matrix)
    P=$1; shift
    timeout 1800 $TR --nproc-per-node $P --master-port $(port) tools/matrix.py --out $OUT/matrix_p$P.jsonl "$@" \
      > $OUT/matrix_p$P.log 2>&1 ;;
  stress)
    P=$1; IT=$2
    timeout 1800 $TR --nproc-per-node $P --master-port $(port) tests/mp_stress_worker.py --iters $IT --layouts all \
      > $OUT/stress_p$P.txt 2>&1 ;;
  ncu-n1)
    timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu "$@" > $OUT/plain.jsonl 2>&1 && \
    timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
      python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu "$@" > $OUT/ncu_launches.log 2>&1 && \
    timeout 1800 ncu --set full --clock-control none --import-source on -k regex:lane_tma_kernel -c 1 \
      -o $OUT/prof python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu "$@" > $OUT/ncu_full.log 2>&1 ;;
  nccl-probe)
    P=$1
    NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,NVLS,TUNING NCCL_DEBUG_FILE=$OUT/nccl_probe_p$P.%h.%p.log \
      timeout 600 $TR --nproc-per-node $P --master-port $(port) tools/nccl_algo_probe.py \
      > $OUT/nccl_probe_p$P.jsonl 2> $OUT/nccl_probe_p$P.err ;;
  *) echo "unknown command $CMD"; exit 2 ;;
esac
