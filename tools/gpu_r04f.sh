timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_batched.py tests/test_gpu_exchange_loopback.py tests/test_gpu_exchange.py tests/test_gpu_psim.py > gpurun_out/r04f_pytest.log 2>&1; tail -1 gpurun_out/r04f_pytest.log
for cfg in "0 1" "1 1" "1 0" "1 2"; do set -- $cfg; TAG="K12=$1 HINT=$2" TLC_K12=$1 TLC_K12_HINT=$2 timeout 300 python tools/k12_probe.py; done > gpurun_out/r04f_probe.txt 2>&1
cat gpurun_out/r04f_probe.txt
for cfg in "0 1" "1 1" "1 2"; do set -- $cfg
  echo "K12=$1 HINT=$2 $(TLC_K12=$1 TLC_K12_HINT=$2 timeout 300 python tools/xchg_w1_once.py 2>&1 | tail -1)"
done > gpurun_out/r04f_w1.txt 2>&1
cat gpurun_out/r04f_w1.txt
for k in 0 1; do TLC_K12=$k W=4 timeout 600 python tools/xchg_loopback_once.py 2>&1 | head -1; done > gpurun_out/r04f_loop.txt 2>&1
cat gpurun_out/r04f_loop.txt
