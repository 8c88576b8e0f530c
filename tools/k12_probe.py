"""K12 vs K1 + K2 on a table of CNT tensors of N values each (env; default 64 x 4,194,320: P % 4 == 0,
every tile vectorised): per-kernel device ms per compress (library profiler), REPS compresses.
A driver for ncu DRAM-byte captures of the fused kernel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1802_07389_b200 as T  # noqa: E402

dev = torch.device("cuda", 0)
cnt, n = int(os.environ.get("CNT", "64")), int(os.environ.get("N", "4194320"))
ts = [torch.randn(n, device=dev) for _ in range(cnt)]
ctx = T.TensorSet([n] * cnt, dev)
for _ in range(3):
    ctx.compress(ts, 1.9, True)
torch.cuda.synchronize()
T.tlc_prof_enable(True)
T.tlc_prof_collect()
reps = int(os.environ.get("REPS", "5"))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    ctx.compress(ts, 1.9, True)
e1.record()
torch.cuda.synchronize()
pr = T.tlc_prof_collect()
print(os.environ.get("TAG", ""), "compress ms", round(e0.elapsed_time(e1) / reps, 4),
      {k: round(v[1] / reps, 4) for k, v in pr.items()}, flush=True)
