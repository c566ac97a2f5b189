# round 2 (bk), 2 GPUs: P = 8 (4 ranks per GPU) at BASELINE configs[1..3] full sizes and every layout at 1 GiB,
# whole-buffer verified through the multi-process path (tools/p8_fullsize_check.py); correctness only.
O=gpurun_out/r2bk; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1"
export LANE_TEST_GPUS=2
timeout 120 $TR --master-port 29961 tools/p8_fullsize_check.py --layouts 2x4 4x2 8x1 1x8 --mib 1024 --calls 2 > $O/p8.txt 2>&1; echo "rc=$?" >> $O/p8.txt
timeout 60 $TR --master-port 29962 tools/p8_fullsize_check.py --layouts 4x2 --k 4 --mib 256 --calls 2 >> $O/p8.txt 2>&1; echo "rc=$?" >> $O/p8.txt
timeout 60 $TR --master-port 29963 tools/p8_fullsize_check.py --layouts 8x1 --dtype bfloat16 --mib 512 --calls 2 >> $O/p8.txt 2>&1; echo "rc=$?" >> $O/p8.txt
