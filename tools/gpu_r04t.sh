# K5m reading a peer's payloads over NVLink, one process on two GPUs: timing, then ncu with the NVLink section
timeout 600 python tools/k5m_nvlink.py > gpurun_out/r04t_k5m_nvlink.txt 2>&1; tail -n 3 gpurun_out/r04t_k5m_nvlink.txt
REPS=1 timeout 900 ncu --set full --section Nvlink --section Nvlink_Tables --import-source on --clock-control none \
  -k regex:"aggregate_par|zre_scan" -s 2 -c 2 -o gpurun_out/r04t_k5m_nvlink -f python tools/k5m_nvlink.py > gpurun_out/r04t_ncu.log 2>&1
tail -n 2 gpurun_out/r04t_ncu.log
