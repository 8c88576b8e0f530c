# A/B of the K2 table kernel's producer warp (TLC_K2T_WS) on the W=1 BERT-large exchange,
# then the large-table and exchange parity tests on the TLC_K2T_WS build.
bash tools/xchg_ab.sh "" "TLC_K2T_WS" "" "TLC_K2T_WS" > gpurun_out/k2t_ws_ab.txt 2>&1
python -c "import __graft_entry__ as g; B=g._builder(); B.build(force=True, defines=('TLC_K2T_WS',))" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_batched.py tests/test_gpu_exchange.py -q -x > gpurun_out/k2t_ws_pytest.log 2>&1
tail -2 gpurun_out/k2t_ws_pytest.log
python -c "import __graft_entry__ as g; B=g._builder(); B.build(force=True)" > /dev/null 2>&1
cat gpurun_out/k2t_ws_ab.txt
