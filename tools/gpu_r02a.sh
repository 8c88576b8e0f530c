# round 2, first GPU call: loopback exchange tests + existing exchange and parity suites
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02a_smoke.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_exchange_loopback.py -q -x > gpurun_out/r02a_loopback.log 2>&1; tail -3 gpurun_out/r02a_loopback.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r02a_pytest_gpu.log 2>&1; tail -3 gpurun_out/r02a_pytest_gpu.log
