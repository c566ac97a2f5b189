# round 2 (y), 4 GPUs: final evidence after the smaller default chunk (512 KiB;
# 256 KiB for one-node layouts): P = 2 chunk check, GPU test tier, N = 1 bench +
# ncu, P = 4 / P = 2 sweeps, bench lines N = 4 / N = 2, configs[4] matrices.
set -x
O=gpurun_out/r2y; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
port=29980
for L in 1x2 2x1; do
  port=$((port+1)); timeout 900 $TR --nproc-per-node 2 --master-port $port tools/tune_mid.py --layout $L --mib 256 1024 --iters 20 \
    --cfg "" "LANE_CHUNK_BYTES=262144" "LANE_CHUNK_BYTES=524288" "LANE_CHUNK_BYTES=1048576" | sed "s/^/$L /" >> $O/tune_p2.txt 2>> $O/tune_p2.err
done
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "rc=$?" >> $O/smoke.txt
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench_n1.jsonl 2> $O/bench_n1.err
bash tools/gpu/lane_gpu.sh r2y ncu-n1
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
