# A/B: lane_emit variant 4 and the K3 literal-list capacity, at s=1.0 / 1.5 / 1.75 and dense
mkdir -p ab
for v in "1 512" "4 512" "4 1024" "4 256"; do set -- $v; python -c "
import importlib.util as u; s=u.spec_from_file_location('b','paper_1802_07389_b200/build.py'); m=u.module_from_spec(s); s.loader.exec_module(m)
m.build(out='ab/e$1c$2.so', defines=['TLC_EMIT_V=$1', 'TLC_K3_LITCAP=$2'])" > /dev/null 2>&1; done
for cfg in "gauss 1.0" "gauss 1.5" "dense 1.75" "gauss 1.75"; do set -- $cfg
  for v in e1c512 e4c512 e4c1024 e4c256; do FAMILY=$1 S=$2 timeout 300 python tools/ab_variants.py ab/$v.so 2>&1 | sed "s/^/$1 s=$2 /"; done
done > gpurun_out/r02p_ab.txt
cat gpurun_out/r02p_ab.txt | sed 's/k1_absmax.*k3_zre/k3_zre/'
