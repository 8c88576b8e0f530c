timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_exchange_loopback.py tests/test_gpu_exchange.py tests/test_gpu_parity.py > gpurun_out/r04o_pytest.log 2>&1; tail -n 1 gpurun_out/r04o_pytest.log
for rep in 1 2; do echo "new $(timeout 300 python tools/xchg_w1_once.py 2>&1 | tail -n 1)"; done > gpurun_out/r04o_w1.txt 2>&1
W=4 timeout 600 python tools/xchg_loopback_once.py 2>&1 | head -n 1 >> gpurun_out/r04o_w1.txt
cat gpurun_out/r04o_w1.txt
