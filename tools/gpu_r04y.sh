TLC_K7_PART=1024 timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_batched.py > gpurun_out/r04y_pytest.log 2>&1; tail -n 1 gpurun_out/r04y_pytest.log
for rep in 1 2; do for v in 2048 1024 4096; do TAG="part=$v" TLC_K7_PART=$v timeout 300 python tools/c2_ab.py; done; done > gpurun_out/r04y_c2.txt 2>&1
cat gpurun_out/r04y_c2.txt
