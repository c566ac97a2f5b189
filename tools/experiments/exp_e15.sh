# 4 GPUs: BASELINE configs[4] matrix at P=4 and P=2 (1 GiB, k in 1,2,4,8, int32+fp32 (+bf16 k=1)), emulated configs[1..3]
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T="timeout 900 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
$T --nproc-per-node=4 --master-port 29881 tools/matrix.py --out gpurun_out/e15_matrix_p4.jsonl > gpurun_out/e15_matrix_p4.log 2>&1
$T --nproc-per-node=4 --master-port 29882 tools/matrix.py --ks 1 --dtypes bfloat16 --out gpurun_out/e15_matrix_p4.jsonl >> gpurun_out/e15_matrix_p4.log 2>&1
$T --nproc-per-node=2 --master-port 29883 tools/matrix.py --out gpurun_out/e15_matrix_p2.jsonl > gpurun_out/e15_matrix_p2.log 2>&1
O=gpurun_out/e15_emu.txt
timeout 120 python tools/quick_time.py --layout 2x4 --k 1 --dtype float32 --mib 1024 >> $O 2>&1
timeout 120 python tools/quick_time.py --layout 4x2 --k 4 --dtype float32 --mib 256 >> $O 2>&1
timeout 120 python tools/quick_time.py --layout 8x1 --k 1 --dtype bfloat16 --mib 512 >> $O 2>&1
timeout 120 python tools/quick_time.py --layout 2x4 --k 1 --dtype float32 --mib 1 >> $O 2>&1
