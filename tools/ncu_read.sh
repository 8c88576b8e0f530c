# summary + per-line instruction counts of a K3/K4 capture made by tools/ncu_k3.sh
rep=gpurun_out/$1.ncu-rep
for k in tlc_zre_kernel tlc_zre_scan_kernel; do ncu -i $rep --page source --csv --kernel-name $k > gpurun_out/src_$k.csv 2>/dev/null; done
ncu -i $rep --page details --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin))
h=r[0]
ki=h.index('Kernel Name'); mi=h.index('Metric Name'); vi=h.index('Metric Value'); ui=h.index('Metric Unit'); ii=h.index('ID')
want=('Duration','Compute (SM) Throughput','Achieved Occupancy','Theoretical Occupancy','Executed Instructions','Issue Slots Busy','Registers Per Thread','Block Limit Shared Mem','Block Limit Registers')
for x in r[1:]:
  if x[mi] in want: print(x[ii],x[ki][:24],x[mi],x[vi],x[ui])
"
d=$(mktemp -d); (cd $d && cuobjdump -xelf compress.sm_100a.cubin /root/repo/gpurun_out/libtlc_cap.so >/dev/null && cuobjdump -xelf decompress.sm_100a.cubin /root/repo/gpurun_out/libtlc_cap.so >/dev/null)
python tools/ncu_lines.py gpurun_out/src_tlc_zre_kernel.csv $d/compress.sm_100a.cubin _ZN3tlc14tlc_zre_kernelENS_8SegTableEPKjfPKhPNS_4CtrlEPy ${2:-30} --outer
python tools/ncu_lines.py gpurun_out/src_tlc_zre_scan_kernel.csv $d/decompress.sm_100a.cubin _ZN3tlc19tlc_zre_scan_kernelENS_8SegTableEPNS_4CtrlEPyS3_ ${3:-15} --outer
