"""The W=1 parameter-server exchange of a model's gradient list (bench.py's xchg_w1 leg) for a
few steps in one process: a driver for ncu captures of the exchange kernels (K5m etc.)."""
import os
import sys
import types

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1802_07389_b200 as T  # noqa: E402

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
args = types.SimpleNamespace(model=os.environ.get("MODEL", "bert-large"), xs=1.9, steps=3, warmup=3,
                             xchg="p2p", no_e2e=True, e2e_steps=0)
r, ms, value = bench.run_exchange_leg(args, T, dev, 1, 0, None, e2e_steps=0)
print("ms", ms, "GB/s", value)
