# round 2 (h), 4 GPUs: programmatic dependent launch (LANE_PDL) and the LL128
# kernel with paired source loads in B/C, vs the build before the LL128 change
# (tools/ab/liblane_pdl.so); steady-state traces with valid ports.
set -x
O=gpurun_out/r2h; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 900 python -m pytest tests/test_gpu_emulated.py -m gpu -x -q -k "ll128 or parity_layouts" > $O/pytest_emulated.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
SIZES="1 2 4 8 16 24 32 64 128"
for rep in 1 2; do
  timeout 900 $TR --master-port 2962$rep tools/tune_mid.py --layout 2x2 --mib $SIZES --iters 50 --cfg "" "LANE_PDL=0" \
    "LANE_PROTO=ll128" "LANE_PROTO=ll128,LANE_PDL=0" >> $O/tune_new.txt 2>&1
  LANE_LIB_PATH=$PWD/tools/ab/liblane_pdl.so timeout 900 $TR --master-port 2963$rep tools/tune_mid.py --layout 2x2 \
    --mib $SIZES --iters 50 --cfg "" "LANE_PROTO=ll128" >> $O/tune_base.txt 2>&1
done
timeout 900 $TR --master-port 29640 tools/tune_mid.py --layout 2x2 --mib 1 4 16 --iters 50 --nccl --cfg "" >> $O/tune_new.txt 2>&1
i=0
for m in 8 16 32; do
  i=$((i+1))
  LANE_PROTO=ll128 timeout 300 $TR --master-port 2965$i tools/trace_run.py --layout 2x2 --mib $m --calls 20 > $O/trace_ll128_${m}.txt 2>&1
done
for m in 32 64; do
  i=$((i+1))
  LANE_PROTO=simple timeout 300 $TR --master-port 2965$i tools/trace_run.py --layout 2x2 --mib $m --calls 20 --register > $O/trace_simple_${m}.txt 2>&1
done
