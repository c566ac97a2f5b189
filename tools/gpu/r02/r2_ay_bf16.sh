# round 2 (ay), 4 GPUs: bf16 busbw vs size (BASELINE configs[3] dtype) on 4x1 (the
# pure-lane shape of configs[3] at P = 4) and 2x2, whole-buffer verified, clocks.
set -x
O=gpurun_out/r2ay; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 1200 $TR --master-port 30951 bench.py --gpus 4 --layout 4x1 --dtype bfloat16 --sweep $O/sweep_bf16_p4.jsonl --mib 512 --nccl-ppg 0 > $O/sweep_4x1.log 2>&1
timeout 1200 $TR --master-port 30952 bench.py --gpus 4 --layout 2x2 --dtype bfloat16 --sweep $O/sweep_bf16_p4.jsonl --mib 512 --nccl-ppg 0 > $O/sweep_2x2.log 2>&1
