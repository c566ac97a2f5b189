# round 2 (i), 4 GPUs: is the per-CTA spread of phase A (identical static
# shares finishing 2x apart) tied to the SM a CTA runs on? Traces with %smid,
# LL128 and simple protocol, 2x2 fp32, two sizes, twice each (stable?).
set -x
O=gpurun_out/r2i; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
i=0
for rep in 1 2; do
for m in 16 32; do
  i=$((i+1))
  LANE_PROTO=ll128 timeout 300 $TR --master-port 2966$i tools/trace_run.py --layout 2x2 --mib $m --calls 20 \
    --dump $O/dump_ll128_${m}_rep${rep}_r%r.jsonl > $O/trace_ll128_${m}_rep$rep.txt 2>&1
done
i=$((i+1))
LANE_PROTO=simple timeout 300 $TR --master-port 2966$i tools/trace_run.py --layout 2x2 --mib 64 --calls 20 --register \
  --dump $O/dump_simple_64_rep${rep}_r%r.jsonl > $O/trace_simple_64_rep$rep.txt 2>&1
done
