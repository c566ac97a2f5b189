# round 2 (bg), 2 GPUs: copy engines trailing an SM push chunk by chunk (tools/ce_ag_micro.cu; DESIGN §11 item 4).
O=gpurun_out/r2bg; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ce_ag_micro tools/ce_ag_micro.cu -lcuda > $O/build.txt 2>&1
timeout 120 /tmp/ce_ag_micro > $O/ce_ag.txt 2>&1; echo "rc=$?" >> $O/ce_ag.txt
