# 1-GPU check after an exchange-path kernel change: gpu tests, W=1 exchange timing + launch list, bench
set -x
timeout 700 python -m pytest tests -m gpu -q -x > gpurun_out/y_pt.log 2>&1; tail -2 gpurun_out/y_pt.log
timeout 300 python tools/xchg_w1_once.py > gpurun_out/y_plain.log 2>&1 || exit 1
tail -1 gpurun_out/y_plain.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/y_launches.csv python tools/xchg_w1_once.py > gpurun_out/y_ncu1.log 2>&1
timeout 400 python bench.py --steps 50 --warmup 5 --cpu-seconds 5 > gpurun_out/y_bench.json 2> gpurun_out/y_bench.err
tail -c 600 gpurun_out/y_bench.json
