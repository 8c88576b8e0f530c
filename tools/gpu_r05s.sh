TLC_K12=1 timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_exchange_loopback.py > gpurun_out/r05s_pytest.log 2>&1; tail -n 1 gpurun_out/r05s_pytest.log
for k in 0 1; do TLC_K12=$k W=4 timeout 600 python tools/xchg_loopback_once.py 2>&1 | head -n 1; TLC_K12=$k W=2 timeout 600 python tools/xchg_loopback_once.py 2>&1 | head -n 1; done
