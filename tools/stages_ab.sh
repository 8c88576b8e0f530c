# A/B of the K2 bulk stage count (TLC_K2_STAGES) on C3 and the W=1 exchange; decoder parity tests first
set -x
timeout 700 python -m pytest tests/test_gpu_parity.py tests/test_gpu_exchange.py tests/test_gpu_batched.py -m gpu -q -x > gpurun_out/s_pt.log 2>&1; tail -2 gpurun_out/s_pt.log
for S in 4 5; do python -c "import __graft_entry__ as g; B=g._builder(); B.build(force=True, out='gpurun_out/lib_st$S.so', defines=('TLC_K2_STAGES=$S',))" > /dev/null 2>&1; done
timeout 300 python tools/ab_variants.py gpurun_out/lib_st4.so gpurun_out/lib_st5.so gpurun_out/lib_st4.so gpurun_out/lib_st5.so 2>&1 | grep -v "^events" > gpurun_out/s_c3.log; cat gpurun_out/s_c3.log
bash tools/xchg_ab.sh "TLC_K2_STAGES=5" "" 2>&1 | grep "^\["
