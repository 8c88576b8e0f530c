# K5m with sources in parallel: loopback parity (all W), aggregate tests, then A/B timings vs the sequential kernel
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_exchange_loopback.py tests/test_gpu_aggregate.py tests/test_gpu_exchange.py -q -x > gpurun_out/r02l_pytest.log 2>&1; tail -2 gpurun_out/r02l_pytest.log
for W in 1 2 3 4 8; do W=$W timeout 300 python tools/xchg_loopback_once.py; TLC_K5M_SEQ=1 W=$W timeout 300 python tools/xchg_loopback_once.py | sed 's/^/SEQ /'; done > gpurun_out/r02l_loopback.txt 2>&1
grep -v status gpurun_out/r02l_loopback.txt
