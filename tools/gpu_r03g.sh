# ncu --set full of K6 (one CTA per tensor) and K6x (CTA pairs) on the C2 batch
set -x
REPS=4 python tools/c2_once.py || exit 1
for v in one pair; do
  if [ $v = one ]; then export TLC_K6_ONE=1; else unset TLC_K6_ONE; fi
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:small_.*compress -s 2 -c 1 \
    -o gpurun_out/r03g_k6_$v -f python tools/c2_once.py > gpurun_out/r03g_ncu_$v.log 2>&1
done
ls -la gpurun_out/
