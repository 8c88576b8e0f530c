# A/B of build variants on the W=1 BERT-large exchange (one GPU): per-kernel ms per step.
# Usage: bash tools/xchg_ab.sh "" "TLC_K2_REALIGN=0" "TLC_K5M_REALIGN=0" ...
for D in "$@"; do
python -c "import __graft_entry__ as g; B=g._builder(); B.build(force=True, defines=tuple(x for x in '$D'.split(',') if x))" > /dev/null 2>&1
for rep in 1 2; do
timeout 300 python - <<PY
import os, sys, types
sys.path.insert(0, os.getcwd())
import torch, bench, paper_1802_07389_b200 as T
dev = torch.device("cuda", 0); torch.cuda.set_device(dev)
args = types.SimpleNamespace(model="bert-large", xs=1.9, steps=20, warmup=5, xchg="p2p", no_e2e=True, e2e_steps=0)
r, ms, value = bench.run_exchange_leg(args, T, dev, 1, 0, None, e2e_steps=0)
print("[$D]", round(ms, 4), {k: round(v["ms_per_step"], 4) for k, v in r["kernels"].items()})
PY
done
done
python -c "import __graft_entry__ as g; B=g._builder(); B.build(force=True)" > /dev/null 2>&1
