# dev experiment (4 GPUs): 2 CTAs per SM for the TMA engine and the LL kernel
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1"
O=gpurun_out/e14_tune.txt
echo "## default build" >> $O
$T --master-port 29871 tools/tune_mid.py --layout 2x2 --mib 1 4 8 16 32 64 256 1024 --iters 20 --cfg "" "LANE_PROTO=ll" >> $O 2>&1
timeout 120 python tools/quick_time.py --layout 2x4 --mib 1024 >> $O 2>&1
echo "## -DLANE_TMA_STAGE_KB=24 -DLANE_TMA_MIN_BLOCKS=2" >> $O
LANE_NVCC_FLAGS="-DLANE_TMA_STAGE_KB=24 -DLANE_TMA_MIN_BLOCKS=2" python -m paper_2508_13397_b200.build --force >> $O 2>&1
$T --master-port 29872 tools/tune_mid.py --layout 2x2 --mib 16 32 64 256 1024 --iters 20 --cfg "LANE_PROTO=simple" "LANE_PROTO=simple,LANE_CTAS_TOTAL=296" >> $O 2>&1
timeout 120 python tools/quick_time.py --layout 2x4 --mib 1024 >> $O 2>&1
echo "## -DLANE_TMA_STAGE_KB=32 -DLANE_TMA_STAGES=3 -DLANE_TMA_MIN_BLOCKS=2" >> $O
LANE_NVCC_FLAGS="-DLANE_TMA_STAGE_KB=32 -DLANE_TMA_STAGES=3 -DLANE_TMA_MIN_BLOCKS=2" python -m paper_2508_13397_b200.build --force >> $O 2>&1
$T --master-port 29873 tools/tune_mid.py --layout 2x2 --mib 16 32 64 256 1024 --iters 20 --cfg "LANE_PROTO=simple,LANE_CTAS_TOTAL=296" >> $O 2>&1
echo "## -DLANE_LL_MIN_BLOCKS=2" >> $O
LANE_NVCC_FLAGS="-DLANE_LL_MIN_BLOCKS=2" python -m paper_2508_13397_b200.build --force >> $O 2>&1
$T --master-port 29874 tools/tune_mid.py --layout 2x2 --mib 1 4 8 16 --iters 20 --cfg "LANE_PROTO=ll" "LANE_PROTO=ll,LANE_LL_CTAS=296" >> $O 2>&1
