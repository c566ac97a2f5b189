# round 2 (be), 2 GPUs: P = 8 ranks through the multi-process path on fewer GPUs
# (8 on one GPU; 4 + 4 on two, peers both local and over NVLink).
set -x
O=gpurun_out/r2be; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 8"
LANE_TEST_GPUS=1 timeout 900 $TR --master-port 29941 tests/mp_samedev_worker.py --quick > $O/samedev_p8_g1.txt 2>&1; echo "rc=$?" >> $O/samedev_p8_g1.txt
LANE_TEST_GPUS=2 timeout 900 $TR --master-port 29942 tests/mp_samedev_worker.py --quick > $O/samedev_p8_g2.txt 2>&1; echo "rc=$?" >> $O/samedev_p8_g2.txt
LANE_TEST_GPUS=2 timeout 600 $TR --master-port 29943 tests/mp_stress_worker.py --iters 300 --layouts all > $O/stress_p8_g2.txt 2>&1; echo "rc=$?" >> $O/stress_p8_g2.txt
LANE_TEST_GPUS=2 timeout 300 $TR --master-port 29944 tests/mp_timeout_worker.py > $O/timeout_p8_g2.txt 2>&1; echo "rc=$?" >> $O/timeout_p8_g2.txt
