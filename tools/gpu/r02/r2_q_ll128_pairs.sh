# round 2 (q), 4 GPUs: LL128 line pairs (15 granules per 256 bytes, 8-byte
# flags): parity (emulated LL128 / ring tests, multi-GPU quick worker, exact
# stress), then A/B vs the 7-granule-line build (tools/ab/liblane_head.so).
set -x
O=gpurun_out/r2q; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
port=29820
timeout 900 python -m pytest tests/test_gpu_emulated.py -m gpu -x -q -k "ll128 or ring" > $O/pytest_ll128_ring.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
port=$((port+1)); timeout 600 $TR --master-port $port tests/mp_worker.py --quick > $O/mp_worker_quick.txt 2>&1
port=$((port+1)); timeout 900 $TR --master-port $port tests/mp_stress_worker.py --iters 2000 --layouts all > $O/stress.txt 2>&1
for rep in 1 2; do
  for L in 2x2 4x1 1x4; do
    port=$((port+1))
    timeout 600 $TR --master-port $port tools/tune_mid.py --layout $L --mib 1 2 4 8 16 24 32 --iters 50 \
      --cfg "LANE_PROTO=ll128" >> $O/ab_new_$L.txt 2>&1
    port=$((port+1))
    LANE_LIB_PATH=$PWD/tools/ab/liblane_head.so timeout 600 $TR --master-port $port tools/tune_mid.py --layout $L \
      --mib 1 2 4 8 16 24 32 --iters 50 --cfg "LANE_PROTO=ll128" >> $O/ab_old_$L.txt 2>&1
  done
done
