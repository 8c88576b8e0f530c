timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_batched.py tests/test_gpu_exchange_loopback.py > gpurun_out/r04e_pytest.log 2>&1; tail -1 gpurun_out/r04e_pytest.log
for cfg in "0 1" "1 1" "2 1" "2 0"; do set -- $cfg; TAG="K12=$1 HINT=$2" TLC_K12=$1 TLC_K12_HINT=$2 timeout 300 python tools/k12_probe.py; done > gpurun_out/r04e_probe.txt 2>&1
cat gpurun_out/r04e_probe.txt
for cfg in "0 1" "1 1" "2 1"; do set -- $cfg
  echo "K12=$1 HINT=$2 $(TLC_K12=$1 TLC_K12_HINT=$2 timeout 300 python tools/xchg_w1_once.py 2>&1 | tail -1)"
done > gpurun_out/r04e_w1.txt 2>&1
cat gpurun_out/r04e_w1.txt
REPS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:absmax_quant_bulk -s 3 -c 1 -o gpurun_out/r04e_k12b -f python tools/k12_probe.py > gpurun_out/r04e_ncu.log 2>&1
tail -1 gpurun_out/r04e_ncu.log
