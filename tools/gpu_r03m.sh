timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_batched.py tests/test_gpu_large_path_small_sizes.py tests/test_gpu_guards.py \
  tests/test_gpu_exchange_loopback.py::test_loopback_matches_oracle > gpurun_out/r03m_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r03m_pytest.log; tail -2 gpurun_out/r03m_pytest.log
for g in 4 8 0; do TAG=g$g TLC_K6G=$g timeout 300 python tools/k6_sizes.py; done > gpurun_out/r03m_sizes.txt 2>&1
cat gpurun_out/r03m_sizes.txt
for cfg in "4 2" "8 2" "4 0" "4 1" "4 3" "0 0"; do set -- $cfg
  TAG="g$1_sub$2" TLC_K6G=$1 TLC_K7_SUB=$2 timeout 300 python tools/c2_ab.py; done > gpurun_out/r03m_c2.txt 2>&1
cat gpurun_out/r03m_c2.txt
for g in 4 8; do for f in 0 1; do echo "== group $g FLUSH=$f"; TLC_K6G=$g MODE=group CASE=c2 FLUSH=$f timeout 300 python tools/k6c_trace.py; done; done > gpurun_out/r03m_trace.txt 2>&1
cat gpurun_out/r03m_trace.txt
