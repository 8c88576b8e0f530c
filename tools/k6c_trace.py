"""Timeline of the small-table compressors (development tool, GPU box): builds a
-DTLC_K6C_TRACE variant of libtlc, compresses the C2 table (ResNet-110, 110 tensors; env
CASE=1x36864 for one 36,864-value tensor) a few times with the L2 flushed before each call
(FLUSH=0: warm), and prints per-phase CTA time distributions in us from the earliest CTA
start of the last call.  MODE=coop (K6c, TLC_COOP=1), one (K6, TLC_K6G=0) or group (K6g,
clusters of $TLC_K6G, default 4)."""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VAR = os.path.join(ROOT, "paper_1802_07389_b200", "libtlc_k6ctrace.so")
if os.environ.get("TLC_LIB") != VAR:
    subprocess.check_call([sys.executable, "-c", "import sys; sys.path.insert(0, %r); "
                           "import importlib.util as u; s = u.spec_from_file_location('b', %r); m = u.module_from_spec(s); "
                           "s.loader.exec_module(m); m.build(out=%r, defines=['TLC_K6C_TRACE'])"
                           % (ROOT, os.path.join(ROOT, "paper_1802_07389_b200", "build.py"), VAR)])
    os.execve(sys.executable, [sys.executable] + sys.argv, dict(os.environ, TLC_LIB=VAR))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1802_07389_b200 as T  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda", 0)
MODE = os.environ.get("MODE", "coop")
sizes = {"c2": synth.RESNET110_SIZES, "1x36864": [36864], "35x36864": [36864] * 35, "1x432": [432], "35x9216": [9216] * 35}[os.environ.get("CASE", "c2")]
mus = synth.layer_means(sizes, 2, 110)
ts = [torch.from_numpy(synth.layer_gradient(n, mus[k], 2, 0, k, 0)).to(dev) for k, n in enumerate(sizes)]
if MODE == "coop":
    os.environ["TLC_COOP"] = "1"
elif MODE == "one":
    os.environ["TLC_K6G"] = "0"
flush_on = os.environ.get("FLUSH", "1") == "1"
ctx = T.TensorSet(sizes, dev)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
for k in range(int(os.environ.get("REPS", "5"))):
    if flush_on:
        flush.fill_(k)
    ctx.compress(ts, 1.75, True)
torch.cuda.synchronize()
L = T.lib()
buf = np.zeros((1024, 8), dtype=np.uint64)
L.tlc_debug_k6c_trace.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
assert L.tlc_debug_k6c_trace(buf.ctypes.data, buf.nbytes) == 0
last = {"coop": 6, "one": 5, "group": 6}[MODE]
sel = buf[:, last] > 0
t = buf[sel][:, :last + 1].astype(np.int64)
if MODE != "coop":                                       # slot 7: the SM the CTA ran on
    sm = buf[sel][:, 7].astype(np.int64)
    per = np.bincount(np.bincount(sm, minlength=148))
    print("SMs used", int((np.bincount(sm, minlength=148) > 0).sum()), "| SMs by CTA count:",
          {k: int(v) for k, v in enumerate(per) if v})
t0 = t[:, 0].min()
rel = (t - t0) / 1e3
names = {"coop": ["start", "A loaded", "keys published", "barrier 1 passed", "B done", "barrier 2 passed", "end"],
         "one": ["start", "loaded + max", "quantized", "rows composed", "prefilled", "end"],
         "group": ["start", "loaded + max", "cluster barrier 1", "quantized", "rows summarised",
                   "cluster barrier 2", "end"]}[MODE]
print(f"CTAs {len(t)}")
for i, nm in enumerate(names):
    print(f"{nm:18s} min {rel[:, i].min():7.2f} med {np.median(rel[:, i]):7.2f} max {rel[:, i].max():7.2f} us")
