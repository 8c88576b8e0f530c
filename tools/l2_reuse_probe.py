"""Does K2 read from L2 when it follows K1 on a working set that fits L2?  48 tensors of
4M values (BERT-large's FFN weights): (a) one batch (K1 over all, then K2 over all: HBM twice),
(b) one tlc_compress per tensor (K1 then K2 on 32 MB of t + err).  Per-kernel device ms per
step from the library's profiler, L2 flushed before each step."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1802_07389_b200 as T  # noqa: E402

dev = torch.device("cuda", 0)
N, n = 48, 4 << 20
ts = [torch.randn(n, device=dev) for _ in range(N)]
errs = [torch.zeros(n, device=dev) for _ in range(N)]
ctx = T.TensorSet([n] * N, dev)
pays = [torch.empty(T.tlc_max_payload_bytes(n), dtype=torch.uint8, device=dev) for _ in range(N)]
hdrs = [torch.empty(32, dtype=torch.uint8, device=dev) for _ in range(N)]
ws = torch.empty(T.tlc_compress_workspace_bytes(n), dtype=torch.uint8, device=dev)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)


def step_a():
    ctx.compress(ts, 1.9, True)


def step_b():
    for k in range(N):
        T.tlc_compress(ts[k], errs[k], 1.9, True, pays[k], hdrs[k], ws)


for name, fn in (("batch", step_a), ("per-tensor", step_b)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    T.tlc_prof_enable(True)
    T.tlc_prof_collect()
    reps = 10
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tot = 0.0
    for _ in range(reps):
        flush.fill_(1)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    pr = T.tlc_prof_collect()
    T.tlc_prof_enable(False)
    print(name, "step ms", round(tot / reps, 4), {k: round(v[1] / reps, 4) for k, v in pr.items()}, flush=True)
