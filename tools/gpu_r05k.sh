timeout 1200 python -m pytest -q -x -m gpu tests/test_gpu_parity.py tests/test_gpu_batched.py tests/test_gpu_exchange_loopback.py tests/test_gpu_exchange.py tests/test_gpu_guards.py > gpurun_out/r05k_pytest.log 2>&1; tail -n 1 gpurun_out/r05k_pytest.log
for rep in 1 2; do echo "$(timeout 300 python tools/xchg_w1_once.py 2>&1 | tail -n 1)"; done > gpurun_out/r05k_w1.txt 2>&1
W=4 timeout 600 python tools/xchg_loopback_once.py 2>&1 | head -n 1 >> gpurun_out/r05k_w1.txt
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-c2 --no-xchg-w1 --no-codecs --no-sweep 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C3', d['value'], d['ms_per_step'], {k: round(v['avg_ms'],4) for k,v in d['kernels'].items()})" >> gpurun_out/r05k_w1.txt
cat gpurun_out/r05k_w1.txt
