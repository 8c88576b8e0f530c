REPS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:absmax_quant_bulk -s 3 -c 1 -o gpurun_out/r04d_k12b -f python tools/k12_probe.py > gpurun_out/r04d_ncu.log 2>&1
tail -2 gpurun_out/r04d_ncu.log
