TLC_K12=1 timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_batched.py tests/test_gpu_exchange_loopback.py::test_loopback_large_contexts tests/test_gpu_exchange_loopback.py::test_loopback_bert_large_full_size_sampled tests/test_gpu_exchange_loopback.py::test_loopback_matches_oracle > gpurun_out/r05r_pytest.log 2>&1; tail -n 1 gpurun_out/r05r_pytest.log
for N in 4194320 4194304; do for k in 0 1; do TAG="N=$N K12=$k" N=$N TLC_K12=$k timeout 300 python tools/k12_probe.py; done; done > gpurun_out/r05r_probe.txt 2>&1
cat gpurun_out/r05r_probe.txt
for k in 0 1; do echo "K12=$k $(TLC_K12=$k timeout 300 python tools/xchg_w1_once.py 2>&1 | tail -n 1)"; done
for k in 0 1; do TLC_K12=$k W=4 timeout 600 python tools/xchg_loopback_once.py 2>&1 | head -n 1; done
