# ncu --set full of K3 (gauss s=1.0 steady) and K4 (dense), current tree
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
cp paper_1802_07389_b200/libtlc.so gpurun_out/libtlc_cap.so
FAMILY=gauss S=1.0 REPS=12 timeout 300 ncu --set full --clock-control none --import-source on -k regex:"zre" -s 20 -c 2 -o gpurun_out/r02e_s1 python tools/k3_family_once.py > gpurun_out/r02e_ncu.log 2>&1
FAMILY=dense S=1.75 REPS=3 timeout 300 ncu --set full --clock-control none --import-source on -k regex:"zre" -s 2 -c 2 -o gpurun_out/r02e_dense python tools/k3_family_once.py > gpurun_out/r02e_ncu2.log 2>&1
tail -2 gpurun_out/r02e_ncu.log
