"""Compress + decompress one C3 family tensor a few times (driver for ncu captures of
K3/K4 on dense / low-s data): FAMILY=dense|gauss|runs|zeros S=1.0 N=2^28 REPS=3."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1802_07389_b200 as T  # noqa: E402
import synth  # noqa: E402

n = int(os.environ.get("N", str(1 << 28)))
fam = os.environ.get("FAMILY", "dense")
s = float(os.environ.get("S", "1.75"))
reps = int(os.environ.get("REPS", "3"))
dev = torch.device("cuda", 0)
ts = [synth.family_torch(fam, n, s, dev, 3, k) for k in range(2)]
err = torch.zeros(n, device=dev)
out = torch.empty(n, device=dev)
for k in range(reps):
    if fam != "gauss":
        err.zero_()
    p, h = T.tlc_compress(ts[k % 2], err, s, True)
    T.tlc_decompress(p, h, n, out)
torch.cuda.synchronize()
print("ok", T.parse_header(h))
