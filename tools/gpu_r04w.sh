for S in 1.75 1.0; do for rep in 1 2; do S=$S timeout 600 python tools/ab_variants.py ab/base.so ab/k4c32768.so ab/k4c65536.so 2>&1 | grep -v events | sed "s/^/s=$S /"; done; done > gpurun_out/r04w_ab.txt 2>&1
cat gpurun_out/r04w_ab.txt | sed 's/k1_absmax.*k3_zre/k3_zre/'
for lib in base k4c65536; do echo "$lib $(TLC_LIB=ab/$lib.so timeout 300 python tools/xchg_w1_once.py 2>&1 | tail -n 1)"; done
TLC_LIB=ab/k4c65536.so timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_parity.py tests/test_gpu_batched.py tests/test_gpu_exchange.py > gpurun_out/r04w_pytest.log 2>&1; tail -n 1 gpurun_out/r04w_pytest.log
