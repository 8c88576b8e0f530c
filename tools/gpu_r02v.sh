# K7 over exact parts, K5m okmask, NCCL exact transport (W=1): tests + C2 and loopback timings
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_exchange_loopback.py tests/test_gpu_batched.py tests/test_gpu_parity.py tests/test_gpu_guards.py tests/test_gpu_aggregate.py -q -x > gpurun_out/r02v_pytest.log 2>&1; tail -2 gpurun_out/r02v_pytest.log
TAG=k6 timeout 300 python tools/c2_ab.py > gpurun_out/r02v_c2.txt 2>&1; cat gpurun_out/r02v_c2.txt
for W in 2 4 8; do W=$W timeout 300 python tools/xchg_loopback_once.py; done 2>&1 | grep -v status | sed 's/k1_absmax.*k5_expand/k5_expand/'
