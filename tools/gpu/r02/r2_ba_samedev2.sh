# round 2 (ba), 1 GPU: P = 2 and P = 4 ranks on one GPU through the multi-GPU code path.
set -x
O=gpurun_out/r2ba; mkdir -p $O
for P in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 3097$P \
    tests/mp_samedev_worker.py > $O/samedev_p$P.txt 2>&1; echo "rc=$?" >> $O/samedev_p$P.txt
done
