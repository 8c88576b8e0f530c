# full GPU suite on 2 GPUs + smoke + N=2 bench (after K6g became the small-table compressor)
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r03u_smoke.log 2>&1; tail -3 gpurun_out/r03u_smoke.log
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r03u_pytest_n2.log 2>&1; tail -3 gpurun_out/r03u_pytest_n2.log
bash tools/gpu_r02_multi.sh r03u
