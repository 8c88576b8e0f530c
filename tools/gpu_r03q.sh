for c in 1x432 1x36864 35x9216; do for mode in group one; do echo "== $mode $c"; MODE=$mode CASE=$c FLUSH=0 timeout 300 python tools/k6c_trace.py; done; done > gpurun_out/r03q_trace.txt 2>&1
cat gpurun_out/r03q_trace.txt
