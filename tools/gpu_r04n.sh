python tools/xchg_w1_once.py > /dev/null 2>&1 || exit 1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:expand_dequant -s 3 -c 1 -o gpurun_out/r04n_apply -f python tools/xchg_w1_once.py > gpurun_out/r04n_ncu.log 2>&1
tail -n 1 gpurun_out/r04n_ncu.log
