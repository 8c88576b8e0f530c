"""B200-native 3LC state-change compression (arXiv 1802.07389) -- Python binding.

Thin ctypes marshalling over the C ABI of ``include/tlc.h`` (``libtlc.so``, built
in-tree from ``csrc/`` for sm_100a).  Functions keep the C names
(``tlc_compress``, ``tlc_decompress``, ...); torch is used only to own device
memory and to supply the CUDA stream.  Every step of the method runs in the
CUDA kernels; there is no CPU fallback -- importing this package without the
built library raises.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtlc.so")

TLC_OK, TLC_ERR_ARG, TLC_ERR_NONFINITE, TLC_ERR_RANGE, TLC_ERR_FORMAT, TLC_ERR_CAPACITY, \
    TLC_ERR_CUDA, TLC_ERR_NCCL = range(8)
TLC_FLAG_ZRE = 1
TLC_MODE_OVERWRITE, TLC_MODE_ACCUMULATE = 0, 1
HEADER_BYTES = 32


class TlcError(RuntimeError):
    def __init__(self, code: int, where: str):
        super().__init__(f"{where}: {tlc_status_string(code)} ({code})")
        self.code = code


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(nvcc, sm_100a). There is no CPU fallback.")
    L = ctypes.CDLL(LIB_PATH)
    P, U64, SZ, F, I = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_size_t, ctypes.c_float, ctypes.c_int
    sig = {
        "tlc_version": (I, []),
        "tlc_status_string": (ctypes.c_char_p, [I]),
        "tlc_quartic_bytes": (U64, [U64]),
        "tlc_max_payload_bytes": (U64, [U64]),
        "tlc_compress_workspace_bytes": (SZ, [U64]),
        "tlc_decompress_workspace_bytes": (SZ, [U64]),
        "tlc_compress": (I, [P, P, U64, F, I, P, U64, P, P, SZ, P]),
        "tlc_decompress": (I, [P, P, U64, P, I, P, SZ, P]),
        "tlc_launch_count": (ctypes.c_ulonglong, []),
        "tlc_prof_enable": (None, [I]),
        "tlc_prof_collect": (I, [P, I]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype, fn.argtypes = res, args
    return L


_lib = _load()


def lib():
    return _lib


# ------------------------------------------------------------------ sizes / strings
def tlc_version() -> int:
    return _lib.tlc_version()


def tlc_status_string(code: int) -> str:
    return _lib.tlc_status_string(int(code)).decode()


def tlc_quartic_bytes(n: int) -> int:
    return int(_lib.tlc_quartic_bytes(n))


def tlc_max_payload_bytes(n: int) -> int:
    return int(_lib.tlc_max_payload_bytes(n))


def tlc_compress_workspace_bytes(n: int) -> int:
    return int(_lib.tlc_compress_workspace_bytes(n))


def tlc_decompress_workspace_bytes(n: int) -> int:
    return int(_lib.tlc_decompress_workspace_bytes(n))


# ------------------------------------------------------------------ helpers
def _stream_ptr(stream) -> int:
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream)


def _check_dev(name, x, dtype):
    if not isinstance(x, torch.Tensor) or not x.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if x.dtype != dtype or not x.is_contiguous():
        raise TypeError(f"{name} must be contiguous {dtype}")


_ws_cache: dict = {}


def workspace(nbytes: int, device=None, tag: str = "default") -> torch.Tensor:
    """A cached device workspace of at least ``nbytes`` (torch allocations are
    >= 512-byte aligned, the ABI needs 256)."""
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    key = (dev, tag)
    w = _ws_cache.get(key)
    if w is None or w.numel() < nbytes:
        w = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=dev)
        _ws_cache[key] = w
    return w


def new_header(device=None) -> torch.Tensor:
    return torch.zeros(HEADER_BYTES, dtype=torch.uint8, device=device or "cuda")


def parse_header(hdr: torch.Tensor) -> dict:
    """Copy a device header to the host (synchronizes) and decode its fields."""
    import struct

    raw = bytes(hdr.detach().to("cpu").numpy().tobytes())
    M, flags, n, plen, status, _ = struct.unpack("<fIQQII", raw)
    return {"M": M, "flags": flags, "n": n, "payload_len": plen, "status": status}


# ------------------------------------------------------------------ the ABI calls
def tlc_compress(t: torch.Tensor, err: torch.Tensor, s: float, use_zre: bool = True,
                 payload: torch.Tensor | None = None, hdr: torch.Tensor | None = None,
                 ws: torch.Tensor | None = None, stream=None):
    """Enqueue 3LC compression of ``t`` with error buffer ``err`` (updated in place).
    Returns (payload, hdr) device tensors; read lengths/status with parse_header()."""
    _check_dev("t", t, torch.float32)
    _check_dev("err", err, torch.float32)
    n = t.numel()
    if err.numel() != n:
        raise ValueError("err must have as many elements as t")
    cap = tlc_max_payload_bytes(n)
    if payload is None:
        payload = torch.empty(max(cap, 1), dtype=torch.uint8, device=t.device)
    if hdr is None:
        hdr = new_header(t.device)
    need = tlc_compress_workspace_bytes(n)
    if ws is None:
        ws = workspace(need, t.device, "compress")
    rc = _lib.tlc_compress(t.data_ptr(), err.data_ptr(), n, ctypes.c_float(s), int(bool(use_zre)),
                           payload.data_ptr(), payload.numel(), hdr.data_ptr(), ws.data_ptr(),
                           ws.numel(), _stream_ptr(stream))
    if rc != TLC_OK:
        raise TlcError(rc, "tlc_compress")
    return payload, hdr


def tlc_decompress(payload: torch.Tensor, hdr: torch.Tensor, n: int, out: torch.Tensor | None = None,
                   mode: int = TLC_MODE_OVERWRITE, ws: torch.Tensor | None = None, stream=None):
    """Enqueue decompression into ``out`` (fp32[n]); mode ACCUMULATE adds M*q where q != 0."""
    if out is None:
        out = torch.empty(n, dtype=torch.float32, device=payload.device)
    _check_dev("out", out, torch.float32)
    _check_dev("payload", payload, torch.uint8)
    _check_dev("hdr", hdr, torch.uint8)
    need = tlc_decompress_workspace_bytes(n)
    if ws is None:
        ws = workspace(need, out.device, "decompress")
    rc = _lib.tlc_decompress(payload.data_ptr(), hdr.data_ptr(), n, out.data_ptr(), int(mode),
                             ws.data_ptr(), ws.numel(), _stream_ptr(stream))
    if rc != TLC_OK:
        raise TlcError(rc, "tlc_decompress")
    return out


# ------------------------------------------------------------------ instrumentation
class _ProfEntry(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char_p), ("launches", ctypes.c_ulonglong), ("total_ms", ctypes.c_double)]


def tlc_launch_count() -> int:
    return int(_lib.tlc_launch_count())


def tlc_prof_enable(on: bool = True) -> None:
    _lib.tlc_prof_enable(int(bool(on)))


def tlc_prof_collect() -> dict:
    """{kernel name: (launches, total device ms)} since the last collect (synchronizes)."""
    arr = (_ProfEntry * 16)()
    k = _lib.tlc_prof_collect(ctypes.cast(arr, ctypes.c_void_p), 16)
    return {arr[i].name.decode(): (int(arr[i].launches), float(arr[i].total_ms)) for i in range(min(k, 16))}


compress = tlc_compress
decompress = tlc_decompress
