# round 2 (bi), 1 GPU: host-buffer API tests after the binding's stream/device fix, smoke, short N=1 bench.
O=gpurun_out/r2bi; mkdir -p $O
timeout 300 python -m pytest tests -m gpu -q -k "host" > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "rc=$?" >> $O/smoke.txt
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu > $O/bench.jsonl 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
