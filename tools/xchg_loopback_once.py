"""The parameter-server exchange of a model's gradient set with W virtual ranks on ONE GPU
(tlc_loopback_*): push + pull REPS times, then per-kernel device times of one more step
(library events).  Driver for ncu captures of K5m at W > 1 and for A/B of the exchange
kernels without a multi-GPU box.  Env: MODEL (bert-large | resnet50 | resnet110), W, S, REPS."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1802_07389_b200 as T  # noqa: E402
import synth  # noqa: E402

model = os.environ.get("MODEL", "bert-large")
W = int(os.environ.get("W", "4"))
s = float(os.environ.get("S", "1.9"))
reps = int(os.environ.get("REPS", "3"))
dev = torch.device("cuda", 0)
sizes = synth.MODELS[model]
g = T.Loopback(W, sizes, dev)
grads = [synth.model_step_torch(model, 0, r, dev) for r in range(W)]
outs = [[torch.zeros(n, device=dev) for n in sizes] for _ in range(W)]
for k in range(reps):
    g.push(grads, s)
    g.pull(outs, s)
torch.cuda.synchronize()
T.tlc_prof_collect()
T.tlc_prof_enable(True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
g.push(grads, s)
g.pull(outs, s)
e1.record()
torch.cuda.synchronize()
T.tlc_prof_enable(False)
prof = T.tlc_prof_collect()
print(f"{model} W={W} s={s}: step (all {W} ranks, serialised on one GPU) {e0.elapsed_time(e1):.3f} ms; "
      + "  ".join(f"{k}={v[1]:.4f}ms/{v[0]}" for k, v in prof.items()), flush=True)
print("status", [x.status() for x in g.ranks])
