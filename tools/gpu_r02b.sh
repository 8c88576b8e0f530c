# K3 dense-row staging: parity suites, then the default bench line (with the C3 sweep)
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02b_smoke.log 2>&1
# (parity suites ran green in the first r02b call)
timeout 900 python bench.py > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err; tail -c 1500 gpurun_out/r02b_bench.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r02b_bench.json").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], d["roofline"]["frac"], d["clocks"])
for r in d["c3_sweep"]["runs"]:
    print(r["label"], round(r["value"],1), round(r["ms_per_step"],4), round(r["bits_per_value"],3), round(r["step_alg_frac"],3), {k: v["avg_ms"] for k, v in r["kernels"].items()})
for c in d["next3_codecs"]["designs"]:
    print(c["design"], round(c["value"], 1), c["kernel_ms"])
PY
