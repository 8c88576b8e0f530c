"""K1 then K2 on one 4M-value tensor (32 MB of t + err): ncu's DRAM bytes of K2 show whether
it reads the data K1 just read from L2 (driver for ncu --metrics dram__bytes_read.sum)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1802_07389_b200 as T  # noqa: E402

dev = torch.device("cuda", 0)
n = int(os.environ.get("N", str(4 << 20)))
t = torch.randn(n, device=dev)
err = torch.zeros(n, device=dev)
for _ in range(4):
    T.tlc_compress(t, err, 1.9, True)
torch.cuda.synchronize()
print("ok")
