python tools/xchg_w1_once.py > /dev/null 2>&1 || exit 1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"expand_dequant_kernel<1>|zre_scan|aggregate" -s 6 -c 4 -o gpurun_out/r04j_xchg -f python tools/xchg_w1_once.py > gpurun_out/r04j_ncu.log 2>&1
tail -1 gpurun_out/r04j_ncu.log
