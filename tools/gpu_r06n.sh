# round-end rehearsal on one GPU: build + smoke, full pytest -m gpu, default bench (timed by wall clock too)
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r06n_smoke.log 2>&1; tail -2 gpurun_out/r06n_smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r06n_pytest.log 2>&1; tail -2 gpurun_out/r06n_pytest.log
s=$(date +%s); timeout 1200 python bench.py > gpurun_out/r06n_bench.json 2> gpurun_out/r06n_bench.err; echo "bench rc=$? wall=$(( $(date +%s) - s ))s"
s=$(date +%s); timeout 1200 python bench.py --impl reference > gpurun_out/r06n_ref.json 2> gpurun_out/r06n_ref.err; echo "ref rc=$? wall=$(( $(date +%s) - s ))s"
