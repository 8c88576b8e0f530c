# A/B: K3 register budget (TLC_K3_MINB 3: smem already limits K3 to 3 CTAs/SM) x lane_emit variant
mkdir -p ab
for v in "1 4" "1 3" "2 3" "3 3" "4 3"; do set -- $v; python -c "
import importlib.util as u; s=u.spec_from_file_location('b','paper_1802_07389_b200/build.py'); m=u.module_from_spec(s); s.loader.exec_module(m)
m.build(out='ab/e$1m$2.so', defines=['TLC_EMIT_V=$1', 'TLC_K3_MINB=$2'])" > /dev/null 2>&1; done
for cfg in "gauss 1.0" "dense 1.75" "gauss 1.75" "gauss 1.5"; do set -- $cfg
  for v in e1m4 e1m3 e2m3 e3m3 e4m3; do FAMILY=$1 S=$2 timeout 300 python tools/ab_variants.py ab/$v.so 2>&1 | sed "s/^/$1 s=$2 /"; done
done > gpurun_out/r02x_ab.txt
cat gpurun_out/r02x_ab.txt | sed 's/k1_absmax.*k3_zre/k3_zre/; s/k4_zre.*//'
