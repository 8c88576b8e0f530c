"""A/B of the C2 (ResNet-110) step: compress + decompress of the 110-tensor batch in a CUDA
graph, L2 flushed before each step; prints the mean step time in us."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1802_07389_b200 as T  # noqa: E402

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
for s in (1.0, 1.75):
    r = bench.measure_resnet110(T, dev, s, steps=100)
    print(os.environ.get("TAG", ""), s, round(r["ms_per_step"] * 1e3, 1), round(r["warm"]["ms_per_step"] * 1e3, 1),
          r["kernel_us_cold"], flush=True)
