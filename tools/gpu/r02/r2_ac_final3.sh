# round 2 (ac), 4 GPUs: final evidence with dynamic chunk claims (auto) — GPU
# test tier + smoke, P = 4 / P = 2 sweeps (Alg. 1 ring and approach 2 on 2x2),
# bench lines N = 4 (self-launch) / N = 2 (torchrun), configs[4] matrices, stress.
set -x
O=gpurun_out/r2ac; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "rc=$?" >> $O/smoke.txt
port=30040
port=$((port+1)); timeout 1200 $TR --nproc-per-node 4 --master-port $port bench.py --gpus 4 --layout 2x2 --sweep $O/sweep_p4.jsonl --mib 1024 --ring --approach2 > $O/sweep_p4_2x2.log 2>&1
for L in 4x1 1x4; do
  port=$((port+1)); timeout 1200 $TR --nproc-per-node 4 --master-port $port bench.py --gpus 4 --layout $L --sweep $O/sweep_p4.jsonl --mib 1024 > $O/sweep_p4_$L.log 2>&1
done
for L in 1x2 2x1; do
  port=$((port+1)); timeout 1200 $TR --nproc-per-node 2 --master-port $port bench.py --gpus 2 --layout $L --sweep $O/sweep_p2.jsonl --mib 1024 > $O/sweep_p2_$L.log 2>&1
done
timeout 1200 python bench.py --gpus 4 --steps 20 --warmup 5 > $O/bench_n4.jsonl 2> $O/bench_n4.err
port=$((port+1)); timeout 1200 $TR --nproc-per-node 2 --master-port $port bench.py --gpus 2 --steps 20 --warmup 5 > $O/bench_n2.jsonl 2> $O/bench_n2.err
port=$((port+1)); timeout 1500 $TR --nproc-per-node 4 --master-port $port tools/matrix.py --out $O/matrix_p4.jsonl --dtypes float32 int32 bfloat16 > $O/matrix_p4.log 2>&1
port=$((port+1)); timeout 1500 $TR --nproc-per-node 2 --master-port $port tools/matrix.py --out $O/matrix_p2.jsonl --dtypes float32 int32 > $O/matrix_p2.log 2>&1
port=$((port+1)); timeout 1200 $TR --nproc-per-node 4 --master-port $port tests/mp_stress_worker.py --iters 3000 --layouts all > $O/stress_p4.txt 2>&1
