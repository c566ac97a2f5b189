# dev experiment (4 GPUs): steady-state traces, default sweep, P=4 bench line
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1"
port=29770
for spec in "2x2 16 20" "4x1 16 20" "2x2 1024 5"; do
 set -- $spec; port=$((port+1))
 echo "### $1 $2 MiB steady state ($3 calls)" >> gpurun_out/e7_trace.txt
 $T --master-port $port tools/trace_run.py --layout $1 --mib $2 --calls $3 2>/dev/null | grep -v "^\*\|OMP" >> gpurun_out/e7_trace.txt
done
$T --master-port 29790 bench.py --gpus 4 > gpurun_out/e7_bench_n4.jsonl 2> gpurun_out/e7_bench_n4.err
export BENCH_ARGS="--ring"
bash tools/sweep_sizes.sh 4 2x2 1024 gpurun_out/e7_sizes.txt ""
