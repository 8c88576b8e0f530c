timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_batched.py tests/test_gpu_large_path_small_sizes.py tests/test_gpu_guards.py > gpurun_out/r03r_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r03r_pytest.log; tail -2 gpurun_out/r03r_pytest.log
for cfg in "4 2" "4 1" "0 1"; do set -- $cfg; TAG="g$1b$2" TLC_K6G=$1 TLC_K6G_BULK=$2 timeout 300 python tools/k6_sizes.py; done > gpurun_out/r03r_sizes.txt 2>&1
cat gpurun_out/r03r_sizes.txt
for c in 1x432 35x9216 c2; do echo "== group b2 $c"; MODE=group CASE=$c FLUSH=0 timeout 300 python tools/k6c_trace.py; done > gpurun_out/r03r_trace.txt 2>&1
cat gpurun_out/r03r_trace.txt
