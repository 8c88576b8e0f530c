# PDL on the exchange path and the codec step: A/B by TLC_PDL (loopback W=4, bench W=1 exchange and C3 step)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for rep in 1 2; do for P in 0 1; do TLC_PDL=$P W=4 timeout 300 python tools/xchg_loopback_once.py | sed "s/^/PDL=$P /"; done; done 2>&1 | grep step | sed 's/k1_absmax.*k5_expand/k5_expand/'
for rep in 1 2; do for P in 0 1; do TLC_PDL=$P timeout 600 python bench.py --steps 20 --no-e2e --no-c2 --no-cpu-baseline --no-codecs --no-sweep > gpurun_out/r02z_b$P.json 2>/dev/null; python - $P <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/r02z_b{sys.argv[1]}.json").read().strip().splitlines()[-1])
print("PDL", sys.argv[1], "C3", round(d["ms_per_step"], 4), "xchg_w1", round(d["xchg_w1"]["ms_per_step"], 4))
PY
done; done
