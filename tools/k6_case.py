"""One size list (env CASE: a key of tools/k6_sizes.py's cases) compressed REPS times eagerly
-- a driver for ncu captures of K6 on one workload."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1802_07389_b200 as T  # noqa: E402
import synth  # noqa: E402

cases = {"c2": synth.RESNET110_SIZES, "1x36864": [36864], "1x432": [432], "35x36864": [36864] * 35}
sizes = cases[os.environ.get("CASE", "1x36864")]
dev = torch.device("cuda", 0)
ts = [torch.randn(n, device=dev) for n in sizes]
ctx = T.TensorSet(sizes, dev)
b = ctx.compress_batch(ts)
for _ in range(int(os.environ.get("REPS", "4"))):
    b.compress(1.75, True)
torch.cuda.synchronize()
print("ok")
