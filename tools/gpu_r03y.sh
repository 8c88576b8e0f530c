python tools/xchg_w1_once.py > /dev/null 2>&1 || exit 1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:absmax_quant -s 2 -c 1 -o gpurun_out/r03y_k12 -f python tools/xchg_w1_once.py > gpurun_out/r03y_ncu.log 2>&1
TLC_K12=0 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"absmax|quant_qe" -c 12 --csv --log-file gpurun_out/r03y_k1k2.csv python tools/xchg_w1_once.py > /dev/null 2>&1
tail -2 gpurun_out/r03y_ncu.log
