# W=1 exchange (BERT-large): gpu tests, plain timing, launch list, ncu --set full of K2 table / K5m / K5
set -x
timeout 700 python -m pytest tests -m gpu -q -x > gpurun_out/x_pt.log 2>&1; tail -2 gpurun_out/x_pt.log
timeout 300 python tools/xchg_w1_once.py > gpurun_out/x_plain.log 2>&1 || exit 1
tail -1 gpurun_out/x_plain.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/x_launches.csv python tools/xchg_w1_once.py > gpurun_out/x_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"quant_qe_bulk_table|aggregate|expand_dequant" -s 18 -c 3 -o gpurun_out/x_full python tools/xchg_w1_once.py > gpurun_out/x_ncu2.log 2>&1
