"""Run the desk-scale simulator (paper_1802_07389_b200/psim.py) for the paper's designs and
write a JSON summary: per design final loss / test accuracy and average bits per state change
of pushes and pulls (Table 2's accounting), plus the per-step push / pull bits
trace (the shape of Fig. size-sm).  Usage: python tools/psim_sweep.py out.json"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1802_07389_b200 import psim  # noqa: E402

DESIGNS = [("32-bit float", dict(codec="none")), ("8-bit int", dict(codec="int8")),
           ("Stoch 3-value + QE", dict(codec="stoch", use_zre=False)),
           ("3LC s=1.00 (no ZRE)", dict(codec="3lc", s=1.0, use_zre=False))] + \
          [(f"3LC s={s:.2f}", dict(codec="3lc", s=s)) for s in (1.0, 1.5, 1.75, 1.9)]


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/psim.json"
    steps = int(os.environ.get("PSIM_STEPS", "600"))
    torch.cuda.set_device(0)
    res = []
    for name, kw in DESIGNS:
        t0 = time.time()
        cfg = psim.SimConfig(workers=4, steps=steps, eval_every=100, **kw)
        log = psim.Sim(cfg).run()
        summ = psim.summarize(log)
        stride = max(1, steps // 60)
        res.append({"design": name, **summ, "seconds": time.time() - t0,
                    "trace": [[r["step"], round(r["bits_per_value_push"], 4), round(r["bits_per_value_pull"], 4),
                               round(r["loss"], 4)] for r in log[::stride]]})
        print(name, {k: (round(v, 4) if isinstance(v, float) else v) for k, v in summ.items()}, flush=True)
    cfg = psim.SimConfig(workers=4, steps=steps)
    with open(out, "w") as f:
        json.dump({"config": {k: getattr(cfg, k) for k in cfg.__dataclass_fields__ if k not in ("codec", "s", "use_zre")},
                   "task": "synthetic Gaussian blobs (synth.blobs), 1-hidden-layer MLP, W=4 virtual workers, one server",
                   "designs": res}, f, indent=1)


if __name__ == "__main__":
    main()
