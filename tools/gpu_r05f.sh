timeout 1500 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_ddp_hook.py tests/test_gpu_multidevice.py -q > gpurun_out/r05f_pytest_n2.log 2>&1; tail -n 1 gpurun_out/r05f_pytest_n2.log
for k in 0 1; do TLC_NO_KEYED=$k timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2951$k bench.py --gpus 2 --steps 20 --warmup 5 --no-e2e > gpurun_out/r05f_bench_k$k.json 2> gpurun_out/r05f_bench_k$k.err
python -c "
import json; d=json.loads(open('gpurun_out/r05f_bench_k$k.json').read().strip().splitlines()[-1]); print('NO_KEYED=$k', d['value'], d['ms_per_step'], {k: round(v['ms_per_step'],4) for k,v in d['kernels_rank0'].items()})"; done
