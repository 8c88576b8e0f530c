"""Run each compared-design codec (and the 3LC codec) on the bench tensor a few times: a small
driver for ncu captures (tools: ncu -k regex:... python tools/codec_once.py)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1802_07389_b200 as T  # noqa: E402
import synth  # noqa: E402

n = int(os.environ.get("N", str(1 << 28)))
reps = int(os.environ.get("REPS", "3"))
t = torch.from_numpy(synth.gaussian(n, 3, 0)).cuda()
err = torch.zeros_like(t)
out = torch.empty_like(t)
for k in range(reps):
    p, h = T.tlc_stoch_compress(t, 7, k, False)
    T.tlc_decompress(p, h, n, out)
    c, h8 = T.tlc_int8_compress(t)
    T.tlc_int8_decompress(c, h8, n, out)
    p, h = T.tlc_compress(t, err, 1.75, True)
    T.tlc_decompress(p, h, n, out)
torch.cuda.synchronize()
print("ok")
