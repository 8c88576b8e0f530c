"""CPU oracle of 3LC's compression pipeline (arXiv 1802.07389, Sec. 3) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
``paper_1802_07389_b200`` never imports it, and the two share no code: the
arithmetic lives in ``oracle/tlc_oracle.c`` (plain C, fp32, one IEEE op per
source operation, see its header) and this module only marshals numpy arrays
into it.  ``exchange.py`` holds the W-virtual-rank parameter-server simulation
(X1-X6 in DESIGN.md) built from these calls.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tlc_oracle.c")
_LIB = os.path.join(_HERE, "libtlc_oracle.so")
_LIB_OMP = os.path.join(_HERE, "libtlc_oracle_omp.so")

# Status values (defined independently of include/tlc.h).
OK, ERR_ARG, ERR_NONFINITE, ERR_RANGE, ERR_FORMAT = 0, 1, 2, 3, 4

CFLAGS = ["-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off", "-fno-fast-math"]


def build(force: bool = False, omp: bool = False) -> str:
    """Compile tlc_oracle.c with gcc (no FMA contraction, no fast-math); omp=True builds
    the same source with -fopenmp (element-wise loops on all host cores, bench.py's
    cpu_baseline only)."""
    out = _LIB_OMP if omp else _LIB
    if force or not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(_SRC):
        tmp = out + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, *(["-fopenmp"] if omp else []), "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, out)
    return out


_lib = None
_omp = False


def use_openmp(on: bool) -> None:
    """Switch the functions below to the -fopenmp build (True) or the plain one."""
    global _lib, _omp
    if bool(on) != _omp:
        _omp, _lib = bool(on), None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build(omp=_omp))
        P, U64, F, I = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_float, ctypes.c_int
        sig = {
            "tlc_o_accumulate": (None, [P, P, U64, P]),
            "tlc_o_scale": (I, [P, U64, F, P, P]),
            "tlc_o_quantize": (None, [P, U64, F, P]),
            "tlc_o_dequantize": (None, [P, U64, F, P]),
            "tlc_o_residual": (None, [P, P, U64, F, P]),
            "tlc_o_quartic_len": (U64, [U64]),
            "tlc_o_quartic_encode": (None, [P, U64, P]),
            "tlc_o_quartic_decode": (I, [P, U64, U64, P]),
            "tlc_o_zre_encode": (U64, [P, U64, P]),
            "tlc_o_zre_decode": (I, [P, U64, P, U64]),
            "tlc_o_compress": (I, [P, P, U64, F, I, P, U64, P, P]),
            "tlc_o_decompress": (I, [P, U64, I, F, U64, P, I]),
            "tlc_o_philox4x32_10": (None, [P, P, P]),
            "tlc_o_stoch_word": (ctypes.c_uint32, [U64, U64, U64]),
            "tlc_o_stoch_quantize": (I, [P, U64, U64, U64, P, P]),
            "tlc_o_stoch_compress": (I, [P, U64, U64, U64, I, P, U64, P, P]),
            "tlc_o_int8_compress": (I, [P, U64, P, P]),
            "tlc_o_int8_decompress": (None, [P, U64, F, P, I]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _f32(a) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float32)
    return a


# --------------------------------------------------------------------------- steps
def accumulate(t, buf):
    t, buf = _f32(t), _f32(buf)
    u = np.empty_like(t)
    lib().tlc_o_accumulate(_p(t), _p(buf), t.size, _p(u))
    return u


def scale(u, s):
    """Eq. 1 over u; returns (status, M, max|u|)."""
    u = _f32(u)
    M, a = ctypes.c_float(0), ctypes.c_float(0)
    st = lib().tlc_o_scale(_p(u), u.size, ctypes.c_float(s), ctypes.byref(M), ctypes.byref(a))
    return st, np.float32(M.value), np.float32(a.value)


def quantize(u, M):
    u = _f32(u)
    q = np.empty(u.size, dtype=np.int8)
    lib().tlc_o_quantize(_p(u), u.size, ctypes.c_float(M), _p(q))
    return q


def dequantize(q, M):
    q = np.ascontiguousarray(q, dtype=np.int8)
    out = np.empty(q.size, dtype=np.float32)
    lib().tlc_o_dequantize(_p(q), q.size, ctypes.c_float(M), _p(out))
    return out


def residual(u, q, M):
    u = _f32(u)
    q = np.ascontiguousarray(q, dtype=np.int8)
    buf = np.empty_like(u)
    lib().tlc_o_residual(_p(u), _p(q), u.size, ctypes.c_float(M), _p(buf))
    return buf


def quartic_len(n: int) -> int:
    return int(lib().tlc_o_quartic_len(n))


def quartic_encode(q):
    q = np.ascontiguousarray(q, dtype=np.int8)
    out = np.empty(quartic_len(q.size), dtype=np.uint8)
    lib().tlc_o_quartic_encode(_p(q), q.size, _p(out))
    return out


def quartic_decode(B, n):
    B = np.ascontiguousarray(B, dtype=np.uint8)
    q = np.empty(n, dtype=np.int8)
    st = lib().tlc_o_quartic_decode(_p(B), B.size, n, _p(q))
    return st, q


def zre_encode(B):
    B = np.ascontiguousarray(B, dtype=np.uint8)
    Z = np.empty(max(B.size, 1), dtype=np.uint8)
    z = lib().tlc_o_zre_encode(_p(B), B.size, _p(Z))
    return Z[:z].copy()


def zre_decode(Z, P):
    Z = np.ascontiguousarray(Z, dtype=np.uint8)
    B = np.empty(max(P, 1), dtype=np.uint8)
    st = lib().tlc_o_zre_decode(_p(Z), Z.size, _p(B), P)
    return st, B[:P].copy()


# --------------------------------------------------------------------------- pipeline
class Compressed:
    """Result of compress(): the transmitted pair (payload bytes, M) plus metadata."""

    __slots__ = ("status", "M", "n", "use_zre", "payload")

    def __init__(self, status, M, n, use_zre, payload):
        self.status, self.M, self.n, self.use_zre, self.payload = status, M, n, use_zre, payload

    @property
    def payload_len(self) -> int:
        return int(self.payload.size)


def compress(t, buf, s, use_zre=True):
    """Fig. compression steps 1,2,a,b,3,4.  ``buf`` (np.float32) is updated in place
    on success and untouched on a data error (R6)."""
    t = _f32(t)
    assert isinstance(buf, np.ndarray) and buf.dtype == np.float32 and buf.flags.c_contiguous
    n = t.size
    cap = max(quartic_len(n), 1)
    payload = np.empty(cap, dtype=np.uint8)
    M, ln = ctypes.c_float(0), ctypes.c_uint64(0)
    st = lib().tlc_o_compress(_p(t), _p(buf), n, ctypes.c_float(s), int(bool(use_zre)),
                              _p(payload), cap, ctypes.byref(M), ctypes.byref(ln))
    if st != OK:
        return Compressed(st, np.float32(0), n, use_zre, payload[:0].copy())
    return Compressed(st, np.float32(M.value), n, use_zre, payload[: ln.value].copy())


def decompress(payload, zre_flag, M, n, out=None, accumulate=False):
    """Reverse path; returns (status, out).  accumulate=True adds M*q where q != 0 (R16)."""
    payload = np.ascontiguousarray(payload, dtype=np.uint8)
    if out is None:
        out = np.zeros(n, dtype=np.float32)
    assert out.dtype == np.float32 and out.flags.c_contiguous and out.size == n
    pb = payload if payload.size else np.zeros(1, dtype=np.uint8)
    st = lib().tlc_o_decompress(_p(pb), payload.size, int(bool(zre_flag)), ctypes.c_float(M), n,
                                _p(out), int(bool(accumulate)))
    return st, out


def roundtrip(t, buf, s, use_zre=True):
    c = compress(t, buf, s, use_zre)
    st, out = decompress(c.payload, use_zre, c.M, c.n)
    return c, out


# --------------------------------------------------------------------------- compared designs (Sec. 5.1)
def philox4x32_10(ctr, key):
    """Philox4x32-10 block (Random123): four 32-bit counter words, two key words."""
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.empty(4, dtype=np.uint32)
    lib().tlc_o_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def stoch_word(seed: int, step: int, e: int) -> int:
    """The random word of element e at (seed, step) (reading R22)."""
    return int(lib().tlc_o_stoch_word(seed, step, e))


def stoch_quantize(t, seed: int, step: int):
    """Stochastic 3-value quantization; returns (status, m, q)."""
    t = _f32(t)
    q = np.empty(t.size, dtype=np.int8)
    m = ctypes.c_float(0)
    st = lib().tlc_o_stoch_quantize(_p(t), t.size, seed, step, _p(q), ctypes.byref(m))
    return st, np.float32(m.value), q


def stoch_compress(t, seed: int, step: int, use_zre=False):
    """"Stoch 3-value + QE": stochastic trits, quartic encoding, optional ZRE.
    Decoded by decompress(payload, use_zre, M, n)."""
    t = _f32(t)
    n = t.size
    cap = max(quartic_len(n), 1)
    payload = np.empty(cap, dtype=np.uint8)
    M, ln = ctypes.c_float(0), ctypes.c_uint64(0)
    st = lib().tlc_o_stoch_compress(_p(t), n, seed, step, int(bool(use_zre)), _p(payload), cap,
                                    ctypes.byref(M), ctypes.byref(ln))
    if st != OK:
        return Compressed(st, np.float32(0), n, use_zre, payload[:0].copy())
    return Compressed(st, np.float32(M.value), n, use_zre, payload[: ln.value].copy())


def int8_compress(t):
    """"8-bit int"; returns (status, scale, codes int8[n])."""
    t = _f32(t)
    codes = np.empty(max(t.size, 1), dtype=np.int8)
    sc = ctypes.c_float(0)
    st = lib().tlc_o_int8_compress(_p(t), t.size, _p(codes), ctypes.byref(sc))
    return st, np.float32(sc.value), codes[: t.size].copy()


def int8_decompress(codes, scale, out=None, accumulate=False):
    codes = np.ascontiguousarray(codes, dtype=np.int8)
    if out is None:
        out = np.zeros(codes.size, dtype=np.float32)
    assert out.dtype == np.float32 and out.flags.c_contiguous and out.size == codes.size
    lib().tlc_o_int8_decompress(_p(codes), codes.size, ctypes.c_float(scale), _p(out), int(bool(accumulate)))
    return out
