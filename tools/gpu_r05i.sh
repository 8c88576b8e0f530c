for cfg in "gauss 1.0" "gauss 1.75" "dense 1.75"; do set -- $cfg; for rep in 1 2; do FAMILY=$1 S=$2 timeout 600 python tools/ab_variants.py ab/base.so ab/nopad.so 2>&1 | grep -v events | sed "s/^/$1 s=$2 /"; done; done > gpurun_out/r05i_ab.txt 2>&1
cat gpurun_out/r05i_ab.txt | sed 's/k1_absmax.*k3_zre/k3_zre/; s/k4_zre.*//'
TLC_LIB=ab/nopad.so timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_parity.py tests/test_gpu_batched.py > gpurun_out/r05i_pytest.log 2>&1; tail -n 1 gpurun_out/r05i_pytest.log
