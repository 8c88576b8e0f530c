# 2-GPU validation: full gpu tests (W = 2 exchange included), W=1 launch list, N=1 and N=2 bench lines
set -x
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/z_pt.log 2>&1; tail -2 gpurun_out/z_pt.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/z_launches.csv python tools/xchg_w1_once.py > gpurun_out/z_ncu1.log 2>&1
timeout 400 python bench.py --steps 50 --warmup 5 --cpu-seconds 5 > gpurun_out/z_bench.json 2> gpurun_out/z_bench.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --steps 50 --warmup 5 > gpurun_out/z_bench_n2.json 2> gpurun_out/z_bench_n2.err
tail -c 300 gpurun_out/z_bench_n2.json
