# multi-GPU evidence of the current tree: full suite + smoke + exchange/DDP + bench at N
N=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r06c_smoke_n$N.log 2>&1; tail -n 1 gpurun_out/r06c_smoke_n$N.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r06c_pytest_all_n$N.log 2>&1; tail -n 1 gpurun_out/r06c_pytest_all_n$N.log
bash tools/gpu_r02_multi.sh r06c
# A/B on the same box: the consumers run K4 again (TLC_NO_PRODSEEK=1)
TLC_NO_PRODSEEK=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29518 bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/r06c_bench_noprodseek_n$N.json 2> gpurun_out/r06c_bench_noprodseek_n$N.err
python - $N <<'PY'
import json, sys
for tag in ("r06c_bench", "r06c_bench_noprodseek"):
    d = json.loads(open(f"gpurun_out/{tag}_n{sys.argv[1]}.json").read().strip().splitlines()[-1])
    print(tag, d["value"], d["ms_per_step"], d.get("speedup_vs_allreduce"), d["resnet50"]["ms_per_step"], d["resnet50"]["speedup_vs_allreduce"])
PY
