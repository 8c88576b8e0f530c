FAMILY=gauss S=1.0 python tools/k3_family_once.py > /dev/null 2>&1 || exit 1
FAMILY=gauss S=1.0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"tlc_zre_kernel" -s 2 -c 1 -o gpurun_out/r05b_k3 -f python tools/k3_family_once.py > gpurun_out/r05b_ncu.log 2>&1
tail -n 1 gpurun_out/r05b_ncu.log
