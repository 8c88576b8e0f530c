timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r05m_bench_n2.json 2> gpurun_out/r05m_bench_n2.err; echo rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/r05m_bench_n2.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['speedup_vs_allreduce'])
r=d['resnet50']; print('r50', r['ms_per_step'], r['value'], r['allreduce_fp32_ms_per_step'], r['speedup_vs_allreduce'], r['status'], {k: round(v['ms_per_step'],4) for k,v in r['kernels_rank0'].items()})"
tail -n 3 gpurun_out/r05m_bench_n2.err
