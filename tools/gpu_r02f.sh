# K6c cooperative small-table compressor: parity (batched, loopback, K6 fallback), C2 timing A/B, ncu of K6c/K6/K7
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_batched.py tests/test_gpu_exchange_loopback.py tests/test_gpu_large_path_small_sizes.py -q -x > gpurun_out/r02f_pytest.log 2>&1; tail -2 gpurun_out/r02f_pytest.log
TLC_COOP=1 TAG=coop timeout 300 python tools/c2_ab.py > gpurun_out/r02f_c2.txt 2>&1
TAG=k6 timeout 300 python tools/c2_ab.py >> gpurun_out/r02f_c2.txt 2>&1
cat gpurun_out/r02f_c2.txt
cp paper_1802_07389_b200/libtlc.so gpurun_out/libtlc_cap.so
REPS=8 timeout 300 ncu --set full --clock-control none --import-source on -k regex:"small" -s 6 -c 2 -o gpurun_out/r02f_c2 python tools/c2_once.py > gpurun_out/r02f_ncu.log 2>&1
TLC_NO_COOP=1 REPS=8 timeout 300 ncu --set full --clock-control none --import-source on -k regex:"small_compress" -s 3 -c 1 -o gpurun_out/r02f_c2k6 python tools/c2_once.py > gpurun_out/r02f_ncu2.log 2>&1
tail -2 gpurun_out/r02f_ncu.log
