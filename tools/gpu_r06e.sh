# the apply's K5 loading the next tile's header and seek entries one tile ahead: default build (3 CTAs/SM,
# 32 B of stack) and TLC_K5A_MINB=2 (127 registers, no stack) vs TLC_K5_NOPF (this tile's, beside the
# header); exchange tests on both prefetch builds, then the N-GPU bench interleaved, same box
N=$(nvidia-smi -L | wc -l)
timeout 600 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_exchange_loopback.py tests/test_gpu_parity.py -q -x > gpurun_out/r06e_pytest_n$N.log 2>&1; tail -1 gpurun_out/r06e_pytest_n$N.log
TLC_LIB=$PWD/ab/libtlc_k5a2.so timeout 600 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_exchange_loopback.py tests/test_gpu_parity.py -q -x > gpurun_out/r06e_pytest_k5a2_n$N.log 2>&1; tail -1 gpurun_out/r06e_pytest_k5a2_n$N.log
for rep in 1 2; do
  for v in pf k5a2 nopf; do
    if [ $v = pf ]; then unset TLC_LIB; else export TLC_LIB=$PWD/ab/libtlc_$v.so; fi
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$rep bench.py --gpus $N --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r06e_bench_${v}${rep}_n$N.json 2> gpurun_out/r06e_bench_${v}${rep}_n$N.err
    python - gpurun_out/r06e_bench_${v}${rep}_n$N.json $v <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[2], round(d["ms_per_step"], 4), "resnet50", round(d["resnet50"]["ms_per_step"], 4), {k: round(v["ms_per_step"], 4) for k, v in d["kernels_rank0"].items()})
PY
  done
done
unset TLC_LIB
