# Multi-GPU evidence: exchange tests and the bench line at N GPUs.  Usage: bash tools/gpu_n.sh <N> <tag>
N=$1; tag=$2
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_ddp_hook.py -q -x > gpurun_out/${tag}_pytest_exchange_n$N.log 2>&1; tail -2 gpurun_out/${tag}_pytest_exchange_n$N.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus $N > gpurun_out/${tag}_bench_n$N.json 2> gpurun_out/${tag}_bench_n$N.err
tail -c 300 gpurun_out/${tag}_bench_n$N.err
python - "$tag" "$N" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/{sys.argv[1]}_bench_n{sys.argv[2]}.json").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], d.get("e2e", {}).get("value"))
print(d.get("c4_resnet110"))
PY
