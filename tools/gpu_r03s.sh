TLC_K6G=1 TLC_K6G_BULK=0 timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_batched.py > gpurun_out/r03s_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r03s_pytest.log; tail -2 gpurun_out/r03s_pytest.log
for cfg in "1 0" "4 0" "4 1" "0 1"; do set -- $cfg; TAG="g$1b$2" TLC_K6G=$1 TLC_K6G_BULK=$2 timeout 300 python tools/k6_sizes.py; done > gpurun_out/r03s_sizes.txt 2>&1
cat gpurun_out/r03s_sizes.txt
for cfg in "1 0" "4 0"; do set -- $cfg; for c in 1x432 35x9216; do echo "== group g$1 b$2 $c"; TLC_K6G=$1 TLC_K6G_BULK=$2 MODE=group CASE=$c FLUSH=0 timeout 300 python tools/k6c_trace.py; done; done > gpurun_out/r03s_trace.txt 2>&1
cat gpurun_out/r03s_trace.txt
