timeout 700 python -m pytest tests -m gpu -q -x > gpurun_out/pt.log 2>&1; tail -3 gpurun_out/pt.log
timeout 400 python bench.py --steps 50 --warmup 5 --cpu-seconds 5 > gpurun_out/b.json 2> gpurun_out/b.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/b.json").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], d["bits_per_value"])
print({k: round(v["avg_ms"], 4) for k, v in d["kernels"].items()})
for c in d["c2_resnet110"] or []:
    print(c["s"], c["ms_per_step"], c["kernel_us_cold"])
print(d["xchg_w1"])
PY
