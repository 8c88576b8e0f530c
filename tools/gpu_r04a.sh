for cfg in "0 4 0" "1 4 1" "1 2 1" "1 1 1" "1 4 2" "1 2 2" "1 1 2" "1 8 2"; do set -- $cfg; TAG="K12=$1 WIN=$2 HINT=$3" TLC_K12=$1 TLC_K12_WIN=$2 TLC_K12_HINT=$3 timeout 300 python tools/k12_probe.py; done > gpurun_out/r04a_probe.txt 2>&1
cat gpurun_out/r04a_probe.txt
for cfg in "2 1" "2 2" "4 2"; do set -- $cfg
TLC_K12_WIN=$1 TLC_K12_HINT=$2 REPS=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"absmax" -s 3 -c 1 --csv --log-file gpurun_out/r04a_ncu_$1_$2.csv python tools/k12_probe.py > /dev/null 2>&1
echo "WIN=$1 HINT=$2"; grep -h "dram\|duration" gpurun_out/r04a_ncu_$1_$2.csv | awk -F'","' '{print $(NF-2), $(NF)}'
done
