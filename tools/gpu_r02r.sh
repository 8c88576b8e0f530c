# K5m: contiguous tile runs, superset loads, hoisted results; K5 accumulate batched loads: parity + loopback timings
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_exchange_loopback.py tests/test_gpu_aggregate.py tests/test_gpu_exchange.py tests/test_gpu_parity.py tests/test_gpu_guards.py -q -x > gpurun_out/r02r_pytest.log 2>&1; tail -2 gpurun_out/r02r_pytest.log
for S in 1.9 1.0; do for W in 1 2 4 8; do S=$S W=$W timeout 300 python tools/xchg_loopback_once.py; done; done > gpurun_out/r02r_loopback.txt 2>&1
grep -v status gpurun_out/r02r_loopback.txt | sed 's/k1_absmax.*k5_expand/k5_expand/'
