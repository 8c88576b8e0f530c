# the apply K5 (ACCUMULATE) over contiguous tile runs per CTA (value tables rebuilt only on a context change):
# exchange + parity tests, then N-GPU bench A/B against the previous build (ab/libtlc_head.so), interleaved, same box
N=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_exchange_loopback.py tests/test_gpu_ddp_hook.py tests/test_gpu_aggregate.py tests/test_gpu_parity.py tests/test_gpu_psim.py tests/test_gpu_batched.py -q -x > gpurun_out/r06m_pytest_n$N.log 2>&1; tail -1 gpurun_out/r06m_pytest_n$N.log
for rep in 1 2; do
  for v in new old; do
    if [ $v = old ]; then export TLC_LIB=$PWD/ab/libtlc_head.so; else unset TLC_LIB; fi
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2955$rep bench.py --gpus $N --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r06m_bench_${v}${rep}_n$N.json 2> gpurun_out/r06m_bench_${v}${rep}_n$N.err
    python - gpurun_out/r06m_bench_${v}${rep}_n$N.json $v <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[2], round(d["ms_per_step"], 4), "resnet50", round(d["resnet50"]["ms_per_step"], 4), {k: round(v["ms_per_step"], 4) for k, v in d["kernels_rank0"].items()})
PY
  done
done
unset TLC_LIB
