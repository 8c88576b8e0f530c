# One GPU call: full gpu test suite, default bench line, then a launch list and an ncu
# --set full capture of the new codec kernels.  Usage: bash tools/gpu_round.sh <tag>
tag=${1:-r01d}
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/${tag}_pytest_gpu.log 2>&1; tail -3 gpurun_out/${tag}_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; tail -c 600 gpurun_out/${tag}_bench.err
python - "$tag" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/{sys.argv[1]}_bench.json").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], d["roofline"]["frac"], d["clocks"])
for c in (d.get("next3_codecs") or {}).get("designs", []):
    print(c["design"], round(c["value"], 1), round(c["ms_per_step"], 4), c["kernel_ms"], round(c["roofline"]["frac"], 3))
PY
