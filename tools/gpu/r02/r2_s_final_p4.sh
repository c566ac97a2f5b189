# round 2 (s), 4 GPUs: evidence on the final build — full GPU test tier (multi-GPU
# cases included) + smoke, busbw-vs-size sweeps at P = 4 and P = 2 (3 repeats,
# whole-buffer verified, clocks, NCCL ring / x4 PPG / default beside; the paper's
# Alg. 1 ring and approach 2 on 2x2), bench lines at N = 4 (self-launch) and
# N = 2 (torchrun), and the configs[4] matrix at P = 4.
set -x
O=gpurun_out/r2s; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
free -g > $O/free.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "rc=$?" >> $O/smoke.txt
port=29860
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
