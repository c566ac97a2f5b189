# round 2 (am), 4 GPUs: the FULL multi-GPU parity worker (not --quick): every
# P = 4 and P = 2 layout x k in {1,2,4,8,16} x dtype x counts up to 2^24+1 (two
# 64 MiB rounds) x every protocol / job set incl. chunk claims, vs the oracle.
set -x
O=gpurun_out/r2am; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 3000 $TR --nproc-per-node 4 --master-port 30201 tests/mp_worker.py > $O/mp_worker_p4.txt 2>&1; echo "rc=$?" >> $O/mp_worker_p4.txt
timeout 2000 $TR --nproc-per-node 2 --master-port 30202 tests/mp_worker.py > $O/mp_worker_p2.txt 2>&1; echo "rc=$?" >> $O/mp_worker_p2.txt
