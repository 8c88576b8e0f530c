# producer seek entries (K3 writes them, the consumers' K5m / K5 skip K4): exchange parity, then A/B on the loopback
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r06b_smoke.log 2>&1; tail -2 gpurun_out/r06b_smoke.log
timeout 1500 python -m pytest tests/test_gpu_exchange_loopback.py tests/test_gpu_exchange.py tests/test_gpu_aggregate.py tests/test_gpu_ddp_hook.py tests/test_gpu_batched.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/r06b_pytest.log 2>&1; tail -3 gpurun_out/r06b_pytest.log
for rep in 1 2; do
for M in bert-large resnet50; do for W in 2 4; do
  MODEL=$M W=$W S=1.9 REPS=5 timeout 300 python tools/xchg_loopback_once.py 2>&1 | grep -v "^status" | sed "s/^/prodseek   /"
  TLC_NO_PRODSEEK=1 MODEL=$M W=$W S=1.9 REPS=5 timeout 300 python tools/xchg_loopback_once.py 2>&1 | grep -v "^status" | sed "s/^/no-prodseek /"
done; done; done > gpurun_out/r06b_ab.txt 2>&1
cat gpurun_out/r06b_ab.txt | cut -c1-250
