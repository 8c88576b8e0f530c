# ncu of K5m (par, W=4, after the tile-run change) and of K6 / K7 on the ResNet-110 table; bench sweep sanity
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
cp paper_1802_07389_b200/libtlc.so gpurun_out/libtlc_cap.so
W=4 REPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"aggregate" -s 4 -c 1 -o gpurun_out/r02u_par4 python tools/xchg_loopback_once.py > gpurun_out/r02u_ncu1.log 2>&1
REPS=8 timeout 300 ncu --set full --clock-control none --import-source on -k regex:"small" -s 6 -c 2 -o gpurun_out/r02u_c2 python tools/c2_once.py > gpurun_out/r02u_ncu2.log 2>&1
tail -n 1 gpurun_out/r02u_ncu1.log gpurun_out/r02u_ncu2.log
