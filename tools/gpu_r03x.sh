# K12 (fused K1/K2 over L2 windows): parity, then exchange-step A/B
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r03x_pytest.log 2>&1; tail -3 gpurun_out/r03x_pytest.log
for cfg in "0 4 0" "1 4 0" "1 2 0" "1 8 0" "1 16 0" "1 4 1" "1 8 1"; do set -- $cfg
  echo "K12=$1 WIN=$2 HINT=$3 $(TLC_K12=$1 TLC_K12_WIN=$2 TLC_K12_HINT=$3 timeout 300 python tools/xchg_w1_once.py 2>&1 | tail -1)"
done > gpurun_out/r03x_w1.txt 2>&1
cat gpurun_out/r03x_w1.txt
for k in 0 1; do TLC_K12=$k W=4 timeout 600 python tools/xchg_loopback_once.py 2>&1 | head -1; done > gpurun_out/r03x_loop.txt 2>&1
cat gpurun_out/r03x_loop.txt
