timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_batched.py tests/test_gpu_guards.py tests/test_gpu_parity.py > gpurun_out/r04x_pytest.log 2>&1; tail -n 1 gpurun_out/r04x_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -n 1
for rep in 1 2; do for v in 1 0; do TAG="spec=$v" TLC_K7_SPEC=$v timeout 300 python tools/c2_ab.py; done; done > gpurun_out/r04x_c2.txt 2>&1
cat gpurun_out/r04x_c2.txt
