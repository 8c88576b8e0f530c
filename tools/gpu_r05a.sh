# final ncu --set full of the small-table kernels (K6g, K7 records) on the ResNet-110 table
REPS=4 python tools/c2_once.py || exit 1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"small_(group|decompress_rec)" -s 2 -c 2 -o gpurun_out/r05a_c2 -f python tools/c2_once.py > gpurun_out/r05a_ncu.log 2>&1
tail -n 1 gpurun_out/r05a_ncu.log
