# C3 headline A/B on one box: the current build vs the build before the producer seek entries (K3 whole-row
# warp split + seek write check; Seg 8 bytes larger), interleaved
timeout 900 python tools/ab_variants.py ab/libtlc_cur.so ab/libtlc_pre_prodseek.so ab/libtlc_cur.so ab/libtlc_pre_prodseek.so ab/libtlc_cur.so ab/libtlc_pre_prodseek.so > gpurun_out/r06h_c3_ab.txt 2>&1; cat gpurun_out/r06h_c3_ab.txt
