# K5m warp-specialised (producer warp + cp.async windows): parity, then A/B vs the parallel kernel (TLC_K5M_PAR=1)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_exchange_loopback.py tests/test_gpu_aggregate.py tests/test_gpu_exchange.py tests/test_gpu_guards.py -q -x > gpurun_out/r03b_pytest.log 2>&1; tail -2 gpurun_out/r03b_pytest.log
for S in 1.9 1.0; do for W in 2 4 8; do for rep in 1 2; do
  S=$S W=$W timeout 300 python tools/xchg_loopback_once.py | sed "s/^/WS  /"
  TLC_K5M_PAR=1 S=$S W=$W timeout 300 python tools/xchg_loopback_once.py | sed "s/^/PAR /"
done; done; done 2>&1 | grep step | sed 's/k1_absmax.*k5_expand/k5_expand/' | tee gpurun_out/r03b_ab.txt
