# multi-GPU evidence (run with gpurun --gpus N): exchange + DDP tests at world N, bench at N (exchange, all-reduce baseline, C4)
N=$(nvidia-smi -L | wc -l)
TAG=${1:-r02q}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_ddp_hook.py -q > gpurun_out/${TAG}_pytest_n$N.log 2>&1; tail -3 gpurun_out/${TAG}_pytest_n$N.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_n$N.json 2> gpurun_out/${TAG}_bench_n$N.err; tail -c 800 gpurun_out/${TAG}_bench_n$N.err
python - $TAG $N <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/{sys.argv[1]}_bench_n{sys.argv[2]}.json").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], d.get("speedup_vs_allreduce"), d["allreduce_fp32"]["ms_per_step"], d["roofline"]["frac"], d["clocks"])
print({k: round(v["ms_per_step"], 4) for k, v in d["kernels_rank0"].items()})
for c in d["c4_resnet110"]["runs"]:
    print(c)
PY
