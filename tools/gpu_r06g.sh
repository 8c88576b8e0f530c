# launch list (ncu) of the W = 4 loopback exchange (BERT-large, s = 1.9): with producer seek entries no K4 runs
MODEL=bert-large W=4 S=1.9 REPS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r06g_loopback_w4_launches.csv python tools/xchg_loopback_once.py > gpurun_out/r06g_ncu.log 2>&1; echo "ncu rc=$?"
python - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/r06g_loopback_w4_launches.csv")) if len(r) > 10]
hdr = rows[0]; ki = hdr.index("Kernel Name"); vi = hdr.index("Metric Value")
c = collections.Counter(); t = collections.Counter()
for r in rows[1:]:
    name = r[ki].split("(")[0].split("<")[0]
    c[name] += 1; t[name] += float(r[vi].replace(",", ""))
for k in sorted(c, key=lambda k: -t[k]):
    print(f"{k:50s} launches {c[k]:4d}  total {t[k]/1e3:9.1f} us")
PY
