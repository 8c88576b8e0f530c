timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_batched.py > gpurun_out/r05t_pytest.log 2>&1; tail -n 1 gpurun_out/r05t_pytest.log
TLC_PDL=1 timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_batched.py > gpurun_out/r05t_pytest_pdl.log 2>&1; tail -n 1 gpurun_out/r05t_pytest_pdl.log
for rep in 1 2; do for v in 0 1; do TAG="pdl=$v" TLC_PDL=$v timeout 300 python tools/c2_ab.py; done; done > gpurun_out/r05t_c2.txt 2>&1
cat gpurun_out/r05t_c2.txt
