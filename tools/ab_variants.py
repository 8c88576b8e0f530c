"""Development tool: time the compress+decompress step of alternative builds of
libtlc.so (tuning experiments, e.g. -DTLC_K2_MINB=2) on the bench workload.

  python tools/ab_variants.py lib1.so lib2.so ...   (GPU box)

Each variant is loaded with ctypes and driven through the same C ABI as the
product binding; per-kernel device times come from tlc_prof_collect."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402


class Ent(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char_p), ("launches", ctypes.c_ulonglong), ("total_ms", ctypes.c_double)]


def run(path, n=1 << 28, s=None, steps=30, warm=45, keep=False, family=None):
    """family (env FAMILY: gauss | dense | runs | zeros) and s (env S) select the C3 input."""
    s = float(os.environ.get("S", "1.75")) if s is None else s
    family = family or os.environ.get("FAMILY", "gauss")
    L = ctypes.CDLL(path)
    P, U64, SZ = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_size_t
    L.tlc_compress.argtypes = [P, P, U64, ctypes.c_float, ctypes.c_int, P, U64, P, P, SZ, P]
    L.tlc_decompress.argtypes = [P, P, U64, P, ctypes.c_int, P, SZ, P]
    L.tlc_compress_workspace_bytes.restype = SZ
    L.tlc_decompress_workspace_bytes.restype = SZ
    L.tlc_prof_collect.argtypes = [P, ctypes.c_int]
    dev = torch.device("cuda")
    ts = ([torch.from_numpy(synth.gaussian(n, 3, k)).to(dev) for k in range(2)] if family == "gauss" else
          [synth.family_torch(family, n, s, dev, 3, k) for k in range(2)])
    err = torch.zeros(n, device=dev)
    out = torch.empty(n, device=dev)
    cap = (n + 4) // 5
    pay = torch.empty(cap, dtype=torch.uint8, device=dev)
    hdr = torch.zeros(32, dtype=torch.uint8, device=dev)
    wc = torch.empty(L.tlc_compress_workspace_bytes(n), dtype=torch.uint8, device=dev)
    wd = torch.empty(L.tlc_decompress_workspace_bytes(n), dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream().cuda_stream

    def step(k):
        if family != "gauss":
            err.zero_()
        L.tlc_compress(ts[k % 2].data_ptr(), err.data_ptr(), n, s, 1, pay.data_ptr(), cap, hdr.data_ptr(),
                       wc.data_ptr(), wc.numel(), st)
        L.tlc_decompress(pay.data_ptr(), hdr.data_ptr(), n, out.data_ptr(), 0, wd.data_ptr(), wd.numel(), st)

    for k in range(warm):                # the error buffer needs ~40 steps to reach its steady state
        step(k)
    torch.cuda.synchronize()
    arr = (Ent * 16)()
    L.tlc_prof_collect(ctypes.cast(arr, P), 16)
    L.tlc_prof_enable(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(steps):
        step(k)
    e1.record()
    torch.cuda.synchronize()
    L.tlc_prof_enable(0)
    k = L.tlc_prof_collect(ctypes.cast(arr, P), 16)
    ms = e0.elapsed_time(e1) / steps
    per = {arr[i].name.decode(): arr[i].total_ms / arr[i].launches for i in range(k)}
    if keep:
        print("events:", "  ".join(f"{a}={b * 1e3:.1f}us" for a, b in per.items()), flush=True)
        return L
    print(os.path.basename(path), f"step {ms:.4f} ms  fp32-in {4 * n / ms / 1e6:.1f} GB/s  ",
          "  ".join(f"{a}={b:.4f}" for a, b in per.items()), flush=True)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        run(p)
