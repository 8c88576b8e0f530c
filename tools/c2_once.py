"""The C2 workload (BASELINE configs[1]: 110 ResNet-110 tensors, one tlc_batch) compressed and
decompressed eagerly a few times -- a small driver for ncu launch lists of the batched path."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1802_07389_b200 as T  # noqa: E402
import synth  # noqa: E402

s = float(os.environ.get("S", "1.75"))
reps = int(os.environ.get("REPS", "6"))
dev = torch.device("cuda", 0)
sizes = synth.RESNET110_SIZES
mus = synth.layer_means(sizes, 2, 110)
ts = [torch.from_numpy(synth.layer_gradient(n, mus[k], 2, 0, k, 0)).to(dev) for k, n in enumerate(sizes)]
outs = [torch.empty(n, dtype=torch.float32, device=dev) for n in sizes]
ctx = T.TensorSet(sizes, dev)
for k in range(reps):
    ctx.compress(ts, s, True)
    ctx.decompress(outs, T.TLC_MODE_OVERWRITE)
torch.cuda.synchronize()
print("ok", sum(h["payload_len"] for h in ctx.headers()))
