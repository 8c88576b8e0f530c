# padded emission stage (K3, K6c), K6c/K7 rework: parity, K6c trace, C2 A/B, sweep, loopback exchange timings
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_codecs.py tests/test_gpu_batched.py tests/test_gpu_exchange_loopback.py tests/test_gpu_large_path_small_sizes.py -q -x > gpurun_out/r02i_pytest.log 2>&1; tail -2 gpurun_out/r02i_pytest.log
timeout 300 python tools/k6c_trace.py > gpurun_out/r02i_k6c_trace.txt 2>&1; cat gpurun_out/r02i_k6c_trace.txt
TLC_COOP=1 TAG=coop timeout 300 python tools/c2_ab.py > gpurun_out/r02i_c2.txt 2>&1; TAG=k6 timeout 300 python tools/c2_ab.py >> gpurun_out/r02i_c2.txt 2>&1; cat gpurun_out/r02i_c2.txt
for W in 1 2 4 8; do W=$W timeout 300 python tools/xchg_loopback_once.py; done > gpurun_out/r02i_loopback.txt 2>&1; cat gpurun_out/r02i_loopback.txt
timeout 600 python bench.py --steps 20 --no-e2e --no-c2 --no-xchg-w1 --no-cpu-baseline --no-codecs > gpurun_out/r02i_bench.json 2> gpurun_out/r02i_bench.err; tail -c 400 gpurun_out/r02i_bench.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r02i_bench.json").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], d["roofline"]["frac"], d["clocks"])
print({k: round(v["avg_ms"], 4) for k, v in d["kernels"].items()})
for r in d["c3_sweep"]["runs"]:
    print(r["label"], round(r["value"],1), round(r["ms_per_step"],4), round(r["bits_per_value"],3), round(r["step_alg_frac"],3), {k: v["avg_ms"] for k, v in r["kernels"].items()})
PY
