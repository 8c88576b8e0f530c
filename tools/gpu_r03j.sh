unset TLC_K6_ONE
for c in 1x432 1x36864; do
CASE=$c timeout 600 ncu --set full --import-source on --clock-control none --warp-sampling-interval 0 \
  -k regex:small_.*compress -s 2 -c 1 -o gpurun_out/r03j_pair_$c -f python tools/k6_case.py >> gpurun_out/r03j_ncu.log 2>&1
done
tail -3 gpurun_out/r03j_ncu.log
