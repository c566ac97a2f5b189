# round 2 (az), 1 GPU: two ranks on one GPU through the multi-GPU code path (IPC,
# sys flags, handshake) — does time-slicing let it complete, and how fast?
set -x
O=gpurun_out/r2az; mkdir -p $O
nvidia-smi -q -d COMPUTE | grep -i "compute mode" > $O/mode.txt 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 30961 \
  tests/mp_samedev_worker.py > $O/samedev.txt 2>&1; echo "rc=$?" >> $O/samedev.txt
