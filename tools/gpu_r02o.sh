# full -m gpu suite (incl. guard bands and the device-check build), then ncu of K5m (par, W=4) and the K5 apply at s=1.0
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02o_smoke.log 2>&1; tail -1 gpurun_out/r02o_smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02o_pytest_gpu.log 2>&1; tail -3 gpurun_out/r02o_pytest_gpu.log
cp paper_1802_07389_b200/libtlc.so gpurun_out/libtlc_cap.so
W=4 REPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"aggregate" -s 4 -c 1 -o gpurun_out/r02o_par4 python tools/xchg_loopback_once.py > gpurun_out/r02o_ncu1.log 2>&1
S=1.0 W=2 REPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"expand_dequant" -s 2 -c 1 -o gpurun_out/r02o_apply python tools/xchg_loopback_once.py > gpurun_out/r02o_ncu2.log 2>&1
tail -n 2 gpurun_out/r02o_ncu1.log; tail -n 2 gpurun_out/r02o_ncu2.log
