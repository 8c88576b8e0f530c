# A/B of K5m build variants in the N=2 exchange bench (run under gpurun --gpus 2).
# Usage: bash tools/k5m_ab.sh "TLC_K5M_MINB=3" "TLC_K5M_MINB=4" ...
for D in "$@"; do
python -c "import __graft_entry__ as g; B=g._builder(); B.build(force=True, defines=('$D',))" > /dev/null 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$D', round(d['value'],1), d['ms_per_step'], {k: round(v['ms_per_step'],3) for k,v in d['kernels_rank0'].items()})"
done
python -c "import __graft_entry__ as g; B=g._builder(); B.build(force=True)" > /dev/null 2>&1
