"""Timeline of the cooperative small-table compressor K6c (development tool, GPU box):
builds a -DTLC_K6C_TRACE variant of libtlc, compresses the C2 table (ResNet-110, 110
tensors) a few times with the L2 flushed before each call, and prints per-phase CTA time
distributions in us from the earliest CTA start of the last call."""
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
sizes = synth.RESNET110_SIZES
mus = synth.layer_means(sizes, 2, 110)
ts = [torch.from_numpy(synth.layer_gradient(n, mus[k], 2, 0, k, 0)).to(dev) for k, n in enumerate(sizes)]
os.environ.setdefault("TLC_COOP", "1")
ctx = T.TensorSet(sizes, dev)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
for k in range(int(os.environ.get("REPS", "5"))):
    flush.fill_(k)
    ctx.compress(ts, 1.75, True)
torch.cuda.synchronize()
L = T.lib()
buf = np.zeros((1024, 8), dtype=np.uint64)
L.tlc_debug_k6c_trace.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
assert L.tlc_debug_k6c_trace(buf.ctypes.data, buf.nbytes) == 0
t = buf[buf[:, 6] > 0][:, :7].astype(np.int64)
t0 = t[:, 0].min()
rel = (t - t0) / 1e3
names = ["start", "A loaded", "keys published", "barrier 1 passed", "B done", "barrier 2 passed", "end"]
print(f"CTAs {len(t)}")
for i, nm in enumerate(names):
    print(f"{nm:18s} min {rel[:, i].min():7.2f} med {np.median(rel[:, i]):7.2f} max {rel[:, i].max():7.2f} us")
