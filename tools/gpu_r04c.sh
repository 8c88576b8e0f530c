timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_batched.py tests/test_gpu_exchange_loopback.py tests/test_gpu_exchange.py > gpurun_out/r04c_pytest.log 2>&1; tail -2 gpurun_out/r04c_pytest.log
for cfg in "0 1" "1 1" "2 1" "2 0"; do set -- $cfg; TAG="K12=$1 HINT=$2" TLC_K12=$1 TLC_K12_HINT=$2 timeout 300 python tools/k12_probe.py; done > gpurun_out/r04c_probe.txt 2>&1
cat gpurun_out/r04c_probe.txt
for cfg in "0 1" "2 1"; do set -- $cfg
  echo "K12=$1 HINT=$2 $(TLC_K12=$1 TLC_K12_HINT=$2 timeout 300 python tools/xchg_w1_once.py 2>&1 | tail -1)"
done > gpurun_out/r04c_w1.txt 2>&1
cat gpurun_out/r04c_w1.txt
