# round 2 (av), 4 GPUs: final sweeps + bench lines on the final code (graph-capable
# kernels, faster binding): P = 4 / P = 2 sweeps (Alg. 1 ring and approach 2 on
# 2x2), bench N = 4 (self-launch) and N = 2 (torchrun).
set -x
O=gpurun_out/r2av; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
port=30800
port=$((port+1)); timeout 1200 $TR --nproc-per-node 4 --master-port $port bench.py --gpus 4 --layout 2x2 --sweep $O/sweep_p4.jsonl --mib 1024 --ring --approach2 > $O/sweep_p4_2x2.log 2>&1
for L in 4x1 1x4; do
  port=$((port+1)); timeout 1200 $TR --nproc-per-node 4 --master-port $port bench.py --gpus 4 --layout $L --sweep $O/sweep_p4.jsonl --mib 1024 > $O/sweep_p4_$L.log 2>&1
done
for L in 1x2 2x1; do
  port=$((port+1)); timeout 1200 $TR --nproc-per-node 2 --master-port $port bench.py --gpus 2 --layout $L --sweep $O/sweep_p2.jsonl --mib 1024 > $O/sweep_p2_$L.log 2>&1
done
timeout 1200 python bench.py --gpus 4 --steps 20 --warmup 5 > $O/bench_n4.jsonl 2> $O/bench_n4.err
port=$((port+1)); timeout 1200 $TR --nproc-per-node 2 --master-port $port bench.py --gpus 2 --steps 20 --warmup 5 > $O/bench_n2.jsonl 2> $O/bench_n2.err
