"""K5m over NVLink in ONE process on two GPUs (a driver for ncu, which must not profile a
multi-rank command): source 0's payloads on cuda:0, source 1's on cuda:1, the fused aggregate
(tlc_aggregate: K4 over the sources, then K5m) on cuda:0 reading source 1 through peer memory.
The mean is checked bit for bit against the same aggregate with both sources local.  Env MODEL
(bert-large), S (1.9), REPS."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1802_07389_b200 as T  # noqa: E402
import synth  # noqa: E402

assert torch.cuda.device_count() >= 2, "needs two GPUs"
model, s, reps = os.environ.get("MODEL", "bert-large"), float(os.environ.get("S", "1.9")), int(os.environ.get("REPS", "5"))
sizes = synth.MODELS[model]
d0, d1 = torch.device("cuda", 0), torch.device("cuda", 1)
rt = ctypes.CDLL("libcudart.so") if os.path.exists("/usr/local/cuda/lib64/libcudart.so") else None
if rt is None:
    rt = ctypes.CDLL("/usr/local/cuda/lib64/libcudart.so.12")
torch.cuda.set_device(d0)
rc = rt.cudaDeviceEnablePeerAccess(1, 0)
assert rc in (0, 704), f"cudaDeviceEnablePeerAccess: {rc}"        # 704: already enabled
sets = []
for w, d in enumerate((d0, d1)):
    torch.cuda.set_device(d)
    ts = T.TensorSet(sizes, d)
    grads = synth.model_step_torch(model, 0, w, d)
    ts.compress(grads, s, True)
    torch.cuda.synchronize(d)
    del grads
    sets.append(ts)
torch.cuda.set_device(d0)
outs = [torch.empty(n, device=d0) for n in sizes]
remote = T.Aggregate(outs, [(sets[0].payloads, sets[0].hdrs), (sets[1].payloads, sets[1].hdrs)])
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(2):
    remote.run()
torch.cuda.synchronize()
T.tlc_prof_enable(True)
T.tlc_prof_collect()
e0.record()
for _ in range(reps):
    remote.run()
e1.record()
torch.cuda.synchronize()
prof = T.tlc_prof_collect()
T.tlc_prof_enable(False)
ms = e0.elapsed_time(e1) / reps
# the same with source 1's payloads copied to cuda:0
p1 = [p.to(d0) for p in sets[1].payloads]
h1 = sets[1].hdrs.to(d0)
outs_l = [torch.empty(n, device=d0) for n in sizes]
local = T.Aggregate(outs_l, [(sets[0].payloads, sets[0].hdrs), (p1, h1)])
local.run()
torch.cuda.synchronize()
same = all(torch.equal(a.view(torch.int32), b.view(torch.int32)) for a, b in zip(outs, outs_l))
z1 = sum(h["payload_len"] for h in sets[1].headers())
print(f"{model} W=2 aggregate on cuda:0, source 1 over NVLink ({z1 / 1e6:.1f} MB of payload): {ms:.4f} ms per run; "
      + "  ".join(f"{k}={v[1] / reps:.4f}ms" for k, v in prof.items()) + f"; bitwise equal to the local run: {same}",
      flush=True)
assert same
