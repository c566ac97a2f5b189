# round 2 (bd), 1 GPU: host<->device copy ceilings and the host-buffer pipeline's piece size.
O=gpurun_out/r2bd; mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1
nvidia-smi -q | grep -A4 "PCI" | grep -i "gen\|width" | head -12 >> $O/topo.txt
timeout 600 python tools/pcie_micro.py --pieces 8 16 32 64 128 > $O/pcie.txt 2>&1; echo "rc=$?" >> $O/pcie.txt
