# round 2 (an), 4 GPUs: CUDA-graph support (device-side epochs) — full GPU tier
# (emulated graph test, multi-GPU workers with graph replays, stress), then an
# A/B of per-call time vs the build before the change (tools/ab/liblane_pregraph.so).
set -x
O=gpurun_out/r2an; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 2400 python -m pytest tests -m gpu -x -q > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
port=30300
for rep in 1 2; do
  for lib in cur pre; do
    if [ $lib = cur ]; then unset LANE_LIB_PATH; else export LANE_LIB_PATH=$PWD/tools/ab/liblane_pregraph.so; fi
    port=$((port+1))
    timeout 600 $TR --master-port $port tools/tune_mid.py --layout 2x2 --mib 0.25 1 4 16 64 1024 --iters 50 --cfg "" \
      | sed "s/^/$lib /" >> $O/ab.txt 2>> $O/ab.err
  done
done
