timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_batched.py tests/test_gpu_large_path_small_sizes.py tests/test_gpu_guards.py \
  tests/test_gpu_exchange_loopback.py::test_loopback_matches_oracle tests/test_gpu_psim.py > gpurun_out/r03t_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r03t_pytest.log; tail -2 gpurun_out/r03t_pytest.log
TLC_K6G_BULK=0 timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_batched.py > gpurun_out/r03t_pytest_b0.log 2>&1
echo "pytest b0 rc=$?" >> gpurun_out/r03t_pytest_b0.log; tail -1 gpurun_out/r03t_pytest_b0.log
for cfg in "4 1" "4 0" "0 1"; do set -- $cfg; TAG="g$1b$2" TLC_K6G=$1 TLC_K6G_BULK=$2 timeout 300 python tools/k6_sizes.py; done > gpurun_out/r03t_sizes.txt 2>&1
cat gpurun_out/r03t_sizes.txt
for rep in 1 2; do for cfg in "4 1" "4 0" "0 1"; do set -- $cfg; TAG="g$1_b$2" TLC_K6G=$1 TLC_K6G_BULK=$2 timeout 300 python tools/c2_ab.py; done; done > gpurun_out/r03t_c2.txt 2>&1
cat gpurun_out/r03t_c2.txt
