timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_batched.py tests/test_gpu_large_path_small_sizes.py > gpurun_out/r03k_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r03k_pytest.log; tail -2 gpurun_out/r03k_pytest.log
TAG=pair timeout 300 python tools/k6_sizes.py > gpurun_out/r03k_sizes.txt 2>&1
TAG=one TLC_K6_ONE=1 timeout 300 python tools/k6_sizes.py >> gpurun_out/r03k_sizes.txt 2>&1
cat gpurun_out/r03k_sizes.txt
for mode in one pair; do for c in 1x36864 c2; do for f in 0 1; do
  echo "== MODE=$mode CASE=$c FLUSH=$f"; MODE=$mode CASE=$c FLUSH=$f timeout 300 python tools/k6c_trace.py
done; done; done > gpurun_out/r03k_trace.txt 2>&1
cat gpurun_out/r03k_trace.txt
