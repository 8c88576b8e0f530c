timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_batched.py tests/test_gpu_large_path_small_sizes.py tests/test_gpu_guards.py \
  tests/test_gpu_exchange_loopback.py::test_loopback_matches_oracle > gpurun_out/r03p_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r03p_pytest.log; tail -2 gpurun_out/r03p_pytest.log
TLC_K6G_BULK=0 timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_batched.py > gpurun_out/r03p_pytest_nobulk.log 2>&1
echo "pytest nobulk rc=$?" >> gpurun_out/r03p_pytest_nobulk.log; tail -2 gpurun_out/r03p_pytest_nobulk.log
for cfg in "4 1" "4 0" "8 1" "2 1" "0 1"; do set -- $cfg; TAG="g$1b$2" TLC_K6G=$1 TLC_K6G_BULK=$2 timeout 300 python tools/k6_sizes.py; done > gpurun_out/r03p_sizes.txt 2>&1
cat gpurun_out/r03p_sizes.txt
for g in 4 2; do echo "== group $g FLUSH=0"; TLC_K6G=$g MODE=group CASE=c2 FLUSH=0 timeout 300 python tools/k6c_trace.py; done > gpurun_out/r03p_trace.txt 2>&1
cat gpurun_out/r03p_trace.txt
for cfg in "4 1" "0 1"; do set -- $cfg; TAG="g$1_b$2" TLC_K6G=$1 TLC_K6G_BULK=$2 timeout 300 python tools/c2_ab.py; done > gpurun_out/r03p_c2.txt 2>&1
cat gpurun_out/r03p_c2.txt
