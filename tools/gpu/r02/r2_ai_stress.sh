# round 2 (ai), 4 GPUs: exact stress on the final build (LL128 line pairs, chunk
# claims) — 20000 back-to-back calls per layout at P = 4 and P = 2, int32/fp32/bf16
# bit-exact vs the canonical-order sum (the R#25 evidence for the line pairs).
set -x
O=gpurun_out/r2ai; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 2400 $TR --nproc-per-node 4 --master-port 30101 tests/mp_stress_worker.py --iters 20000 --layouts all > $O/stress_p4.txt 2>&1
timeout 1800 $TR --nproc-per-node 2 --master-port 30102 tests/mp_stress_worker.py --iters 20000 --layouts all > $O/stress_p2.txt 2>&1
