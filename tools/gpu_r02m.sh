# K5m parallel-source fix: loopback parity; ncu --set full of both K5m variants at W=8 and W=2 (loopback, BERT-large)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_exchange_loopback.py tests/test_gpu_aggregate.py -q -x > gpurun_out/r02m_pytest.log 2>&1; tail -2 gpurun_out/r02m_pytest.log
cp paper_1802_07389_b200/libtlc.so gpurun_out/libtlc_cap.so
W=8 REPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"aggregate" -s 8 -c 1 -o gpurun_out/r02m_par8 python tools/xchg_loopback_once.py > gpurun_out/r02m_ncu1.log 2>&1
TLC_K5M_SEQ=1 W=8 REPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"aggregate" -s 8 -c 1 -o gpurun_out/r02m_seq8 python tools/xchg_loopback_once.py > gpurun_out/r02m_ncu2.log 2>&1
TLC_K5M_SEQ=1 W=2 REPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"aggregate" -s 2 -c 1 -o gpurun_out/r02m_seq2 python tools/xchg_loopback_once.py > gpurun_out/r02m_ncu3.log 2>&1
tail -2 gpurun_out/r02m_ncu1.log gpurun_out/r02m_ncu2.log gpurun_out/r02m_ncu3.log
