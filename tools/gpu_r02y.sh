# K5m occupancy A/B (launch bounds 3 vs 4 CTAs/SM) on the loopback exchange; DDP world-1 tests
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_ddp_hook.py -q > gpurun_out/r02y_pytest.log 2>&1; tail -2 gpurun_out/r02y_pytest.log
mkdir -p ab
for m in 3 4; do python -c "
import importlib.util as u; s=u.spec_from_file_location('b','paper_1802_07389_b200/build.py'); m=u.module_from_spec(s); s.loader.exec_module(m)
m.build(out='ab/k5p$m.so', defines=['TLC_K5P_MINB=$m'])" > /dev/null 2>&1; done
for W in 2 4 8; do for rep in 1 2; do W=$W timeout 600 python tools/xchg_loopback_ab.py ab/k5p3.so ab/k5p4.so; done; done 2>&1 | sed 's/k1_absmax.*k5_expand/k5_expand/' | tee gpurun_out/r02y_ab.txt
