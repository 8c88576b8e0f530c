# K3/K4 on dense data: parity of the K3 change, then ncu --set full of K3 and K4 on the dense family
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_codecs.py -q -x > gpurun_out/r02c_pytest.log 2>&1; tail -2 gpurun_out/r02c_pytest.log
cp paper_1802_07389_b200/libtlc.so gpurun_out/libtlc_cap.so
FAMILY=dense S=1.75 REPS=3 timeout 300 ncu --set full --clock-control none --import-source on -k regex:"zre" -s 2 -c 2 -o gpurun_out/r02c_dense python tools/k3_family_once.py > gpurun_out/r02c_ncu.log 2>&1
FAMILY=gauss S=1.0 REPS=12 timeout 300 ncu --set full --clock-control none --import-source on -k regex:"zre_kernel" -s 10 -c 1 -o gpurun_out/r02c_s1 python tools/k3_family_once.py > gpurun_out/r02c_ncu2.log 2>&1
tail -2 gpurun_out/r02c_ncu.log
