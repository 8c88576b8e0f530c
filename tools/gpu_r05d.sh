timeout 1200 python -m pytest -q -x -m gpu tests/test_gpu_exchange_loopback.py tests/test_gpu_exchange.py > gpurun_out/r05d_pytest.log 2>&1; tail -n 1 gpurun_out/r05d_pytest.log
for k in 0 1; do TLC_NO_KEYED=$k W=4 timeout 600 python tools/xchg_loopback_once.py 2>&1 | head -n 1; TLC_NO_KEYED=$k W=2 timeout 600 python tools/xchg_loopback_once.py 2>&1 | head -n 1; done > gpurun_out/r05d_loop.txt 2>&1
cat gpurun_out/r05d_loop.txt
