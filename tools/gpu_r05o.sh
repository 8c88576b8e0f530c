MODEL=resnet50 W=2 timeout 300 python tools/xchg_loopback_once.py 2>&1 | head -n 1
MODEL=resnet50 W=2 REPS=2 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"zre_scan" -s 4 -c 2 -o gpurun_out/r05o_k4 -f python tools/xchg_loopback_once.py > gpurun_out/r05o_ncu.log 2>&1
tail -n 1 gpurun_out/r05o_ncu.log
