# apply K5 tile order A/B: grid stride (R=1), cyclic runs of 8 (default) or 32, whole contiguous ranges
# (runs): the W = 1 exchange on one GPU, then the N-GPU exchange bench; exchange + parity tests on R=8
N=$(nvidia-smi -L | wc -l)
timeout 600 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_exchange_loopback.py tests/test_gpu_parity.py tests/test_gpu_psim.py -q -x > gpurun_out/r06o_pytest_n$N.log 2>&1; tail -1 gpurun_out/r06o_pytest_n$N.log
for rep in 1 2; do for v in r1 r8 r32 runs; do
  echo "$v w1 $(TLC_LIB=$PWD/ab/libtlc_$v.so timeout 300 python tools/xchg_w1_once.py 2>&1 | grep '^ms')"
done; done
for v in r1 r8 runs; do
  TLC_LIB=$PWD/ab/libtlc_$v.so timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus $N --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r06o_bench_${v}_n$N.json 2> gpurun_out/r06o_bench_${v}_n$N.err
  python - gpurun_out/r06o_bench_${v}_n$N.json $v <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[2], "N", round(d["ms_per_step"], 4), "resnet50", round(d["resnet50"]["ms_per_step"], 4), {k: round(v["ms_per_step"], 4) for k, v in d["kernels_rank0"].items()})
PY
done
