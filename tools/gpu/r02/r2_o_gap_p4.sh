# round 2 (o), 4 GPUs: where the ~7 us per call outside the CTAs' work goes
# (LL128 2x2, steady state): CTA entry before the PDL wait vs start after it.
set -x
O=gpurun_out/r2o; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
i=0
for pdl in 1 0; do
  for m in 2 16; do
    i=$((i+1))
    LANE_PDL=$pdl LANE_PROTO=ll128 timeout 300 $TR --master-port 2976$i tools/trace_run.py --layout 2x2 --mib $m --calls 50 > $O/trace_ll128_${m}_pdl$pdl.txt 2>&1
  done
done
