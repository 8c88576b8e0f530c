./tools/cluster_probe > gpurun_out/r03i_cluster_probe.txt 2>&1
cat gpurun_out/r03i_cluster_probe.txt
export TLC_K6_ONE=1
CASE=1x36864 python tools/k6_case.py || exit 1
CASE=1x36864 timeout 600 ncu --set full --import-source on --clock-control none --warp-sampling-interval 0 \
  -k regex:small_.*compress -s 2 -c 1 -o gpurun_out/r03i_k6_1x36864 -f python tools/k6_case.py > gpurun_out/r03i_ncu.log 2>&1
CASE=1x432 timeout 600 ncu --set full --import-source on --clock-control none --warp-sampling-interval 0 \
  -k regex:small_.*compress -s 2 -c 1 -o gpurun_out/r03i_k6_1x432 -f python tools/k6_case.py >> gpurun_out/r03i_ncu.log 2>&1
tail -3 gpurun_out/r03i_ncu.log
