# round 2 (bh), 2 GPUs: ce_ag_micro at 256 / 64 / 16 chunks, gated and plain copies.
O=gpurun_out/r2bh; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ce_ag_micro tools/ce_ag_micro.cu -lcuda > $O/build.txt 2>&1
for c in 256 64 16; do timeout 120 /tmp/ce_ag_micro $c >> $O/ce_ag.txt 2>&1; timeout 60 /tmp/ce_ag_micro $c u | grep "ce only" >> $O/ce_ag.txt 2>&1; done
echo "rc=$?" >> $O/ce_ag.txt
