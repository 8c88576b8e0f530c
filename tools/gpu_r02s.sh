# K6 staged emission: small-path parity + C2 timing
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_batched.py tests/test_gpu_parity.py tests/test_gpu_guards.py tests/test_gpu_large_path_small_sizes.py tests/test_gpu_device_checks.py -q -x > gpurun_out/r02s_pytest.log 2>&1; tail -2 gpurun_out/r02s_pytest.log
TAG=k6 timeout 300 python tools/c2_ab.py > gpurun_out/r02s_c2.txt 2>&1; cat gpurun_out/r02s_c2.txt
