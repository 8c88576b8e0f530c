# A/B: K3 literal-list capacity 320 / 384 (4 CTAs/SM by shared memory) vs 512 (3 CTAs/SM), lane_emit variant 1
mkdir -p ab
for c in 512 384 320; do python -c "
import importlib.util as u; s=u.spec_from_file_location('b','paper_1802_07389_b200/build.py'); m=u.module_from_spec(s); s.loader.exec_module(m)
m.build(out='ab/c$c.so', defines=['TLC_K3_LITCAP=$c'])" > /dev/null 2>&1; done
for cfg in "gauss 1.75" "gauss 1.9" "gauss 1.5" "gauss 1.0" "dense 1.75"; do set -- $cfg
  for rep in 1 2; do for c in 512 384 320; do FAMILY=$1 S=$2 timeout 300 python tools/ab_variants.py ab/c$c.so 2>&1 | sed "s/^/$1 s=$2 /"; done; done
done > gpurun_out/r03d_ab.txt
cat gpurun_out/r03d_ab.txt | sed 's/k1_absmax.*k3_zre/k3_zre/; s/k4_zre.*//'
