# ncu --set full of the K3/K4 launches of one steady-state bench step (after 45 warm-up steps)
ncu --set full --clock-control none --import-source on -k regex:"zre" -s 90 -c 2 -o gpurun_out/$1 \
    python bench.py --steps 2 --warmup 45 --no-e2e --no-cpu-baseline --no-c2 --no-xchg-w1 > gpurun_out/ncu.log 2>&1
tail -1 gpurun_out/ncu.log
