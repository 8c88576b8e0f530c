# apply K5: cyclic runs of min(8, tiles per CTA) tiles -- exchange + parity tests, N-GPU bench vs whole
# contiguous ranges (ab/libtlc_runs.so, the previous commit)
N=$(nvidia-smi -L | wc -l)
timeout 600 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_exchange_loopback.py tests/test_gpu_parity.py tests/test_gpu_psim.py tests/test_gpu_ddp_hook.py -q -x > gpurun_out/r06p_pytest_n$N.log 2>&1; tail -1 gpurun_out/r06p_pytest_n$N.log
for v in new runs; do
  if [ $v = runs ]; then export TLC_LIB=$PWD/ab/libtlc_runs.so; else unset TLC_LIB; fi
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus $N --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r06p_bench_${v}_n$N.json 2> gpurun_out/r06p_bench_${v}_n$N.err
  python - gpurun_out/r06p_bench_${v}_n$N.json $v <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[2], "N", round(d["ms_per_step"], 4), "resnet50", round(d["resnet50"]["ms_per_step"], 4), "speedup", round(d["speedup_vs_allreduce"], 3), {k: round(v["ms_per_step"], 4) for k, v in d["kernels_rank0"].items()})
PY
done
unset TLC_LIB
echo "w1 $(timeout 300 python tools/xchg_w1_once.py 2>&1 | grep '^ms')"
