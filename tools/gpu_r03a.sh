# checkpoint: full -m gpu suite + smoke + the default bench line
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r03a_smoke.log 2>&1; tail -1 gpurun_out/r03a_smoke.log
timeout 2700 python -m pytest tests -m gpu -q > gpurun_out/r03a_pytest_gpu.log 2>&1; tail -3 gpurun_out/r03a_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r03a_bench.json 2> gpurun_out/r03a_bench.err; tail -c 300 gpurun_out/r03a_bench.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r03a_bench.json").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], d["roofline"]["frac"], d["clocks"], d["gpu_launches"])
print({k: round(v["avg_ms"], 4) for k, v in d["kernels"].items()})
print("cpu", d["cpu_baseline"]["value"], d["cpu_baseline"]["cores"], "e2e", d["e2e"]["value"])
print("xchg_w1", d["xchg_w1"]["ms_per_step"], d["xchg_w1"]["roofline"]["frac"], d["xchg_w1"]["roofline"].get("step_frac"))
print("c2", [(c["s"], round(c["ms_per_step"]*1e3, 1)) for c in d["c2_resnet110"]])
PY
