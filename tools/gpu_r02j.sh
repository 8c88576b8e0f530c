# K6c with slice records + bulk copies, K7 reorder; aggregate + psim + blob + loopback tests; C2 A/B; trace
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_batched.py tests/test_gpu_exchange_loopback.py tests/test_gpu_large_path_small_sizes.py tests/test_gpu_aggregate.py tests/test_gpu_psim.py tests/test_gpu_parity.py -q -x > gpurun_out/r02j_pytest.log 2>&1; tail -2 gpurun_out/r02j_pytest.log
timeout 300 python tools/k6c_trace.py > gpurun_out/r02j_k6c_trace.txt 2>&1; cat gpurun_out/r02j_k6c_trace.txt
TLC_COOP=1 TAG=coop timeout 300 python tools/c2_ab.py > gpurun_out/r02j_c2.txt 2>&1; TLC_COOP=0 TAG=k6 timeout 300 python tools/c2_ab.py >> gpurun_out/r02j_c2.txt 2>&1; cat gpurun_out/r02j_c2.txt
