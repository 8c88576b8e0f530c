# A/B of the expand_scan warp skip (TLC_K5_WSKIP) on C3 (K5 overwrite) and the W=1 exchange; parity tests first
set -x
timeout 700 python -m pytest tests/test_gpu_parity.py tests/test_gpu_exchange.py tests/test_gpu_batched.py -m gpu -q -x > gpurun_out/w_pt.log 2>&1; tail -2 gpurun_out/w_pt.log
python -c "import __graft_entry__ as g; B=g._builder(); B.build(force=True, out='gpurun_out/lib_ws0.so', defines=('TLC_K5_WSKIP=0',))" > /dev/null 2>&1
python -c "import __graft_entry__ as g; B=g._builder(); B.build(force=True, out='gpurun_out/lib_ws1.so')" > /dev/null 2>&1
timeout 300 python tools/ab_variants.py gpurun_out/lib_ws0.so gpurun_out/lib_ws1.so gpurun_out/lib_ws0.so gpurun_out/lib_ws1.so 2>&1 | grep -v "^events" > gpurun_out/w_c3.log; cat gpurun_out/w_c3.log
bash tools/xchg_ab.sh "TLC_K5_WSKIP=0" "" 2>&1 | grep "^\[" 
