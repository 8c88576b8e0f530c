timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_batched.py tests/test_gpu_large_path_small_sizes.py tests/test_gpu_guards.py \
  tests/test_gpu_exchange_loopback.py::test_loopback_matches_oracle > gpurun_out/r03o_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r03o_pytest.log; tail -2 gpurun_out/r03o_pytest.log
for g in 4 2 8 0; do TAG=g$g TLC_K6G=$g timeout 300 python tools/k6_sizes.py; done > gpurun_out/r03o_sizes.txt 2>&1
cat gpurun_out/r03o_sizes.txt
for g in 4 2 8; do echo "== group $g FLUSH=0"; TLC_K6G=$g MODE=group CASE=c2 FLUSH=0 timeout 300 python tools/k6c_trace.py; done > gpurun_out/r03o_trace.txt 2>&1
echo "== one"; MODE=one CASE=c2 FLUSH=0 timeout 300 python tools/k6c_trace.py >> gpurun_out/r03o_trace.txt 2>&1
cat gpurun_out/r03o_trace.txt
