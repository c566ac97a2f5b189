# Long stress with the LL128 protocol in the size mix (LL <= 1 MiB, LL128 1-16 MiB, simple, bulk), every call exact; then N=1 bench
T="timeout 600 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
echo "# tests/mp_stress_worker.py: 20000 back-to-back int32 allreduces per layout on one comm (k=2), sizes 4 B-24 MiB across the LL / LL128 / simple / bulk thresholds, registered or not, in place or not; every call checked exactly" > gpurun_out/l_stress.txt
for L in 2x2 4x1 1x4; do
  $T --nproc-per-node=4 --master-port 29991 tests/mp_stress_worker.py --iters 20000 --layout $L 2>&1 | grep mp_stress >> gpurun_out/l_stress.txt
done
CUDA_VISIBLE_DEVICES=0,1 $T --nproc-per-node=2 --master-port 29992 tests/mp_stress_worker.py --iters 20000 --layout 1x2 2>&1 | grep mp_stress >> gpurun_out/l_stress.txt
cat gpurun_out/l_stress.txt
CUDA_VISIBLE_DEVICES=0 python bench.py > gpurun_out/l_bench_n1.jsonl 2> gpurun_out/l_bench_n1.err; tail -c 600 gpurun_out/l_bench_n1.jsonl
