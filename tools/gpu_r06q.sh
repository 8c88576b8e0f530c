# final tree, one B200: smoke, full pytest -m gpu, default bench line
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r06q_smoke.log 2>&1; tail -2 gpurun_out/r06q_smoke.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r06q_pytest.log 2>&1; tail -2 gpurun_out/r06q_pytest.log
timeout 600 python bench.py > gpurun_out/r06q_bench.json 2> gpurun_out/r06q_bench.err; echo "bench rc=$?"
