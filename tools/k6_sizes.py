"""Where K6's time goes: the compress of size lists (all of one size, or the C2 list), timed
in a CUDA graph of 20 back-to-back compresses (L2 warm; us per compress)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1802_07389_b200 as T  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda", 0)
cases = {"c2": synth.RESNET110_SIZES, "35x36864": [36864] * 35, "1x36864": [36864], "36x2304": [2304] * 36,
         "35x9216": [9216] * 35, "1x432": [432], "148x36864": [36864] * 148, "110x432": [432] * 110}
for name, sizes in cases.items():
    ts = [torch.randn(n, device=dev) for n in sizes]
    ctx = T.TensorSet(sizes, dev)
    b = ctx.compress_batch(ts)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            b.compress(1.75, True, stream=s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(20):
            b.compress(1.75, True, stream=s)
    for _ in range(3):
        g.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(os.environ.get("TAG", ""), name, round(e0.elapsed_time(e1) * 1e3 / 200, 2), "us", flush=True)
