# final tree at N GPUs: exchange + DDP tests, bench line (exchange, all-reduce baseline, C4, ResNet-50)
bash tools/gpu_r02_multi.sh r06l
