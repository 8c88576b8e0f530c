for rep in 1 2; do
TAG=pair timeout 300 python tools/k6_sizes.py
TAG=one TLC_K6_ONE=1 timeout 300 python tools/k6_sizes.py
done > gpurun_out/r03h_sizes.txt 2>&1
cat gpurun_out/r03h_sizes.txt
