"""Development tool: per-chunk K3 timeline from a -DTLC_K3_TRACE build.

  python tools/k3_trace.py ab/v_trace.so      (GPU box)

Runs the C3 bench workload to steady state, then one compress, and prints the
distribution of the phase durations of the chunks (globaltimer, ns)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ab_variants import run  # noqa: E402


def main(path):
    L = run(path, steps=int(os.environ.get("K3_TRACE_STEPS", "1")), warm=45, keep=True)
    buf = np.zeros((1 << 14, 8), dtype=np.uint64)
    L.tlc_debug_k3_trace.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
    assert L.tlc_debug_k3_trace(buf.ctypes.data, buf.nbytes) == 0
    cta = np.zeros((4096, 2), dtype=np.uint64)
    L.tlc_debug_k3_cta.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
    L.tlc_debug_k3_cta(cta.ctypes.data, cta.nbytes)
    nc = int(np.count_nonzero(cta[:, 0]))
    c = cta[:nc].astype(np.int64)
    valid = buf[:, 5] > 0
    n = int(valid.sum())
    t = buf[valid, :6].astype(np.int64)
    t0 = c[:, 0].min()
    print(f"CTAs {nc}: entry spread {(c[:, 0].max() - t0) / 1e3:.2f} us, first fetch {(t[:, 0].min() - t0) / 1e3:.2f} us, "
          f"last phase 3 {(t[:, 5].max() - t0) / 1e3:.2f} us, last exit {(c[:, 1].max() - t0) / 1e3:.2f} us")
    rel = (t - t0) / 1e3                     # us
    print(f"chunks {n}, kernel span {rel[:, 5].max():.1f} us")
    names = ["fetched", "lookback_done", "tma_done", "phase1_done", "fill_done", "phase3_done"]
    for i, nm in enumerate(names):
        print(f"{nm:14s} min {rel[:, i].min():7.2f} med {np.median(rel[:, i]):7.2f} max {rel[:, i].max():7.2f}")
    d = lambda a, b: t[:, b] - t[:, a]
    for a, b, nm in [(0, 2, "tma wait"), (2, 3, "phase 1"), (0, 1, "lookback"), (3, 4, "B1->fill"),
                     (4, 5, "phase 3"), (0, 5, "chunk total")]:
        x = d(a, b) / 1e3
        print(f"{nm:12s} med {np.median(x):6.2f} p90 {np.percentile(x, 90):6.2f} max {x.max():6.2f} us")
    # timeline by chunk id decile
    buf = buf[valid]
    for q in range(0, n, max(1, n // 10)):
        print(f"chunk {q:5d}: start {rel[q,0]:6.1f} tma {rel[q,2]:6.1f} p1 {rel[q,3]:6.1f} lb {rel[q,1]:6.1f} "
              f"fill {rel[q,4]:6.1f} end {rel[q,5]:6.1f}  sm {buf[q,6]} cta {buf[q,7]}")


if __name__ == "__main__":
    main(sys.argv[1])
