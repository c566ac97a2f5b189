# round 2 (bj), 2 GPUs: P = 8 (4 ranks per GPU) at BASELINE configs[1]'s full size through the
# multi-process path, whole-buffer verified (tools/p8_fullsize_check.py); correctness only.
O=gpurun_out/r2bj; mkdir -p $O
LANE_TEST_GPUS=2 timeout 170 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 \
  --master-port 29951 tools/p8_fullsize_check.py --layouts 2x4 --mib 1024 --calls 1 > $O/p8_fullsize.txt 2>&1
echo "rc=$?" >> $O/p8_fullsize.txt
