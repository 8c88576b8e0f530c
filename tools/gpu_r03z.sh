for cfg in "0 4 0" "1 4 0" "1 8 0" "1 4 1"; do set -- $cfg; TAG="K12=$1 WIN=$2 HINT=$3" TLC_K12=$1 TLC_K12_WIN=$2 TLC_K12_HINT=$3 timeout 300 python tools/k12_probe.py; done > gpurun_out/r03z_probe.txt 2>&1
cat gpurun_out/r03z_probe.txt
REPS=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"absmax|quant_qe" -s 3 -c 3 --csv --log-file gpurun_out/r03z_ncu.csv python tools/k12_probe.py > /dev/null 2>&1
TLC_K12=0 REPS=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"absmax|quant_qe" -s 9 -c 3 --csv --log-file gpurun_out/r03z_ncu0.csv python tools/k12_probe.py > /dev/null 2>&1
grep -h "dram\|duration" gpurun_out/r03z_ncu.csv gpurun_out/r03z_ncu0.csv | cut -d, -f5,12-16 | head -20
