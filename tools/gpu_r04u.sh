timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_multidevice.py tests/test_gpu_batched.py > gpurun_out/r04u_pytest.log 2>&1; tail -n 1 gpurun_out/r04u_pytest.log
bash tools/gpu_r04t.sh
