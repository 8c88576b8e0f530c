# ncu --set full of the K5 launch of one steady-state bench step (after 45 warm-up steps)
ncu --set full --clock-control none --import-source on -k regex:"expand_dequant" -s 45 -c 1 -o gpurun_out/$1 \
    python bench.py --steps 2 --warmup 45 --no-e2e --no-cpu-baseline --no-c2 --no-xchg-w1 > gpurun_out/ncu.log 2>&1
tail -1 gpurun_out/ncu.log
