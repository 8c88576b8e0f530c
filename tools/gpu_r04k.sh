timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_batched.py tests/test_gpu_exchange_loopback.py::test_loopback_matches_oracle tests/test_gpu_guards.py > gpurun_out/r04k_pytest.log 2>&1; tail -1 gpurun_out/r04k_pytest.log
TLC_K6G_SYNC=1 timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_batched.py > gpurun_out/r04k_pytest_sync.log 2>&1; tail -1 gpurun_out/r04k_pytest_sync.log
for cfg in "0 4" "1 4" "0 0"; do set -- $cfg; TAG="sync=$1 g=$2" TLC_K6G_SYNC=$1 TLC_K6G=$2 timeout 300 python tools/k6_sizes.py; done > gpurun_out/r04k_sizes.txt 2>&1
cat gpurun_out/r04k_sizes.txt
for rep in 1 2; do for cfg in "0 4" "1 4" "0 0"; do set -- $cfg; TAG="sync=$1 g=$2" TLC_K6G_SYNC=$1 TLC_K6G=$2 timeout 300 python tools/c2_ab.py; done; done > gpurun_out/r04k_c2.txt 2>&1
cat gpurun_out/r04k_c2.txt
MODE=group CASE=c2 FLUSH=0 timeout 300 python tools/k6c_trace.py > gpurun_out/r04k_trace.txt 2>&1; cat gpurun_out/r04k_trace.txt
