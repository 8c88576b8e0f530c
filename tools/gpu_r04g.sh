for N in 4194320 4194304 1048576; do for k in 0 1; do TAG="N=$N K12=$k" N=$N TLC_K12=$k timeout 300 python tools/k12_probe.py; done; done > gpurun_out/r04g_probe.txt 2>&1
cat gpurun_out/r04g_probe.txt
N=4194304 REPS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:absmax_quant -s 3 -c 1 -o gpurun_out/r04g_k12u -f python tools/k12_probe.py > gpurun_out/r04g_ncu.log 2>&1
tail -1 gpurun_out/r04g_ncu.log
