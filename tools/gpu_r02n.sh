# K5m pass-based parallel expansion: parity (loopback, aggregate, exchange), then loopback A/B timings vs the sequential kernel
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_exchange_loopback.py tests/test_gpu_aggregate.py tests/test_gpu_exchange.py tests/test_gpu_psim.py -q -x > gpurun_out/r02n_pytest.log 2>&1; tail -2 gpurun_out/r02n_pytest.log
for W in 1 2 4 8; do W=$W timeout 300 python tools/xchg_loopback_once.py; TLC_K5M_SEQ=1 W=$W timeout 300 python tools/xchg_loopback_once.py | sed 's/^/SEQ /'; done > gpurun_out/r02n_loopback.txt 2>&1
for S in 1.0; do for W in 2 8; do S=$S W=$W timeout 300 python tools/xchg_loopback_once.py; TLC_K5M_SEQ=1 S=$S W=$W timeout 300 python tools/xchg_loopback_once.py | sed 's/^/SEQ /'; done; done >> gpurun_out/r02n_loopback.txt 2>&1
grep -v status gpurun_out/r02n_loopback.txt | sed 's/k1_absmax.*k5_expand/k5_expand/'
