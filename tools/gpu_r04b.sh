timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r04b_pytest.log 2>&1; tail -3 gpurun_out/r04b_pytest.log
for cfg in "0 1" "1 1" "2 1" "2 0"; do set -- $cfg; TAG="K12=$1 HINT=$2" TLC_K12=$1 TLC_K12_HINT=$2 timeout 300 python tools/k12_probe.py; done > gpurun_out/r04b_probe.txt 2>&1
cat gpurun_out/r04b_probe.txt
for cfg in "0 1" "1 1" "2 1" "2 0"; do set -- $cfg
  echo "K12=$1 HINT=$2 $(TLC_K12=$1 TLC_K12_HINT=$2 timeout 300 python tools/xchg_w1_once.py 2>&1 | tail -1)"
done > gpurun_out/r04b_w1.txt 2>&1
cat gpurun_out/r04b_w1.txt
for k in 0 2; do TLC_K12=$k W=4 timeout 600 python tools/xchg_loopback_once.py 2>&1 | head -1; done > gpurun_out/r04b_loop.txt 2>&1
cat gpurun_out/r04b_loop.txt
