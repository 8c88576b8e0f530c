# multi-GPU evidence of the current tree: full suite + smoke + exchange/DDP + bench at N
N=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r06i_smoke_n$N.log 2>&1; tail -n 1 gpurun_out/r06i_smoke_n$N.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r06i_pytest_all_n$N.log 2>&1; tail -n 1 gpurun_out/r06i_pytest_all_n$N.log
bash tools/gpu_r02_multi.sh r06i
