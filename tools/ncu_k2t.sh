set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/k2t_build.log 2>&1
timeout 300 python tools/xchg_w1_once.py > gpurun_out/k2t_plain.log 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/k2t_launches.csv python tools/xchg_w1_once.py > gpurun_out/k2t_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"quant_qe" -s 12 -c 4 -o gpurun_out/k2t_full python tools/xchg_w1_once.py > gpurun_out/k2t_ncu2.log 2>&1
ls gpurun_out
