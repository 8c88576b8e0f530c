# A/B of the three lane_emit variants (K3 dense-row emission) at s=1.0, dense and s=1.75
mkdir -p ab
for v in 1 2 3; do python -c "
import importlib.util as u; s=u.spec_from_file_location('b','paper_1802_07389_b200/build.py'); m=u.module_from_spec(s); s.loader.exec_module(m)
m.build(out='ab/emit$v.so', defines=['TLC_EMIT_V=$v'])" > /dev/null 2>&1; done
for cfg in "gauss 1.0" "dense 1.75" "gauss 1.75" "gauss 1.5"; do set -- $cfg
  for rep in 1 2; do for v in 1 2 3; do FAMILY=$1 S=$2 timeout 300 python tools/ab_variants.py ab/emit$v.so 2>&1 | sed "s/^/$1 s=$2 /"; done; done
done > gpurun_out/r02h_ab.txt
cat gpurun_out/r02h_ab.txt
