# round 2 (bc), 2 GPUs: full GPU test tier on the final code (1-GPU cases, ranks sharing
# one GPU, real P = 2), smoke, and the P = 2 standard-vs-lane sweep (Alg. 1 ring, approach 2).
set -x
O=gpurun_out/r2bc; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests -m gpu -x -q -rs > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "rc=$?" >> $O/smoke.txt
timeout 600 $TR --nproc-per-node 2 --master-port 29931 bench.py --gpus 2 --layout 1x2 --sweep $O/sweep_p2_std.jsonl \
  --mib 1024 --ring --approach2 > $O/sweep_p2_std.log 2>&1; echo "rc=$?" >> $O/sweep_p2_std.log
