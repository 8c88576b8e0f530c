# K6x (CTA pairs) vs K6 (one CTA per tensor): parity of the small-table paths, then the C2 step A/B
set -x
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_batched.py tests/test_gpu_large_path_small_sizes.py \
  tests/test_gpu_exchange_loopback.py::test_loopback_matches_oracle tests/test_gpu_guards.py > gpurun_out/r03f_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r03f_pytest.log
for rep in 1 2; do
  TAG=pair timeout 300 python tools/c2_ab.py
  TAG=one TLC_K6_ONE=1 timeout 300 python tools/c2_ab.py
done > gpurun_out/r03f_c2.txt 2>&1
cat gpurun_out/r03f_c2.txt; tail -3 gpurun_out/r03f_pytest.log
