# round 2 (b): full GPU test tier on a 4-GPU box (multi-GPU tests included),
# smoke, N=1 bench, N=4 bench through the self-launch path and N=2 via torchrun.
set -x
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2b_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2b_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2b_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/r2b_smoke.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2b_bench_n1.jsonl 2> gpurun_out/r2b_bench_n1.err
timeout 900 python bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r2b_bench_n4.jsonl 2> gpurun_out/r2b_bench_n4.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r2b_bench_n2.jsonl 2> gpurun_out/r2b_bench_n2.err
