# round 2 (ax), 4 GPUs: the paper's processes-per-GPU knob across message sizes —
# k in {1, 2, 4, 8, 16} (CTA groups here), 2x2 and 4x1, 1 MiB - 1 GiB.
set -x
O=gpurun_out/r2ax; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
port=30900
for L in 2x2 4x1; do
  for k in 1 2 4 8 16; do
    port=$((port+1))
    timeout 600 $TR --master-port $port tools/tune_mid.py --layout $L --k $k --mib 1 4 16 64 256 1024 --iters 30 --cfg "" \
      | sed "s/^/$L k=$k /" >> $O/ksweep.txt 2>> $O/ksweep.err
  done
done
