# N=2: exchange tests (incl. exact transport), bench per transport, DDP hook vs all-reduce
N=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_exchange.py -q > gpurun_out/r02w_pytest_n$N.log 2>&1; tail -2 gpurun_out/r02w_pytest_n$N.log
for X in nccl nccl-exact; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29518 bench.py --gpus $N --steps 20 --warmup 5 --xchg $X --no-c2 --no-e2e > gpurun_out/r02w_bench_${X}_n$N.json 2> gpurun_out/r02w_bench_${X}_n$N.err
python - gpurun_out/r02w_bench_${X}_n$N.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], d["ms_per_step"], d["value"], d["wire_bytes_per_rank_per_step"], d["speedup_vs_allreduce"], d["roofline"].get("step_frac"))
PY
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29519 tools/ddp_bench.py > gpurun_out/r02w_ddp_n$N.json 2> gpurun_out/r02w_ddp_n$N.err; tail -1 gpurun_out/r02w_ddp_n$N.json
