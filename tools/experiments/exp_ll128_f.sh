# 1 GPU: ncu of the LL128 kernel (emulated 2x4, 8 and 16 MiB per rank), then the N=1 bench line
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
cat > /tmp/ll_prof.py <<'PY'
import os, sys, torch
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
import paper_2508_13397_b200 as lane
from seeded_inputs import device as sdev
mib = float(sys.argv[1]); algo = sys.argv[2]
n = int(mib * (1 << 20)) // 4
os.environ["LANE_PROTO"] = "ll128"
emu = lane.LaneEmulator(2, 4, 1, device=0)
ins = [sdev.fill(torch.empty(n, dtype=torch.float32, device="cuda"), "float32", "signed", 42, p) for p in range(8)]
outs = [torch.empty_like(t) for t in ins]
f = {"lane": emu.allreduce, "ring": emu.allreduce_ring, "a2": emu.allreduce_approach2}[algo]
for _ in range(5):
    f(outs, ins)
torch.cuda.synchronize(); emu.check(); print("ok", mib, algo, emu.protocol(n, "float32"))
PY
for spec in "8 lane lane_ll128_kernel" "16 lane lane_ll128_kernel"; do
  set -- $spec
  python /tmp/ll_prof.py $1 $2 > gpurun_out/f_plain_$2_$1.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$3 -s 3 -c 1 -o gpurun_out/f_prof_$2_$1 \
      python /tmp/ll_prof.py $1 $2 > gpurun_out/f_ncu_$2_$1.log 2>&1
done
python bench.py > gpurun_out/f_bench_n1.jsonl 2> gpurun_out/f_bench_n1.err; tail -1 gpurun_out/f_bench_n1.jsonl
