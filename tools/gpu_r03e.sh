# round-2 launch list of the C3 step (ncu per-launch time + DRAM bytes), ncu --set full of K2 for roofline.traffic; smoke
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r03e_smoke.log 2>&1; tail -2 gpurun_out/r03e_smoke.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none -c 40 --csv --log-file gpurun_out/r03e_launches_raw.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-c2 --no-xchg-w1 --no-codecs --no-sweep > gpurun_out/r03e_ncu.log 2>&1
tail -n 2 gpurun_out/r03e_ncu.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/r03e_launches_time.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-c2 --no-xchg-w1 --no-codecs --no-sweep > gpurun_out/r03e_ncu2.log 2>&1
tail -n 2 gpurun_out/r03e_ncu2.log
