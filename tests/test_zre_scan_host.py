"""CPU test of the GPU zero-run encoder's scan algebra (no GPU needed).

tests/native/zre_scan_host.cu compiles the __host__ __device__ building blocks of
csrc/tlc_device.cuh as host code and drives them through the K2 decomposition
(chunks, rows of 16-byte thread segments, in-order reductions, carry-in
composition, per-row exclusive scans).  Its output must equal the oracle's zero-run encoding byte for byte."""
import ctypes
import os
import subprocess

import numpy as np
import pytest

import oracle as O
import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "native", "zre_scan_host.cu")
LIB = os.path.join(ROOT, "tests", "native", "libzre_scan_host.so")
DEPS = [SRC, os.path.join(ROOT, "paper_1802_07389_b200", "csrc", "tlc_device.cuh")]


@pytest.fixture(scope="module")
def sim():
    if not os.path.exists(LIB) or any(os.path.getmtime(d) > os.path.getmtime(LIB) for d in DEPS):
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-std=c++17", "-O2", "-x", "cu",
                               "-gencode", "arch=compute_100a,code=sm_100a",
                               "-Xcompiler", "-fPIC", "-shared", "-o", LIB, SRC])
    L = ctypes.CDLL(LIB)
    L.zre_scan_sim.restype = ctypes.c_uint64
    L.zre_scan_sim.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint64, ctypes.c_void_p]
    L.zre_scan_sim_mode.restype = ctypes.c_uint64
    L.zre_scan_sim_mode.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint64,
                                    ctypes.c_void_p, ctypes.c_int]

    def run(B, threads, nchunks, lane_mode=0):
        B = np.ascontiguousarray(B, dtype=np.uint8)
        out = np.full(B.size + 16, 0xEE, dtype=np.uint8)
        z = L.zre_scan_sim_mode(B.ctypes.data, B.size, threads, nchunks, out.ctypes.data, lane_mode)
        assert np.all(out[z:] == 0xEE), "bytes emitted past the computed payload length"
        return out[:z]

    run.lib = L
    return run


def _streams():
    g = synth.rng(71)
    yield np.full(1, 121, np.uint8)
    yield np.array([5], np.uint8)
    for L in (13, 14, 15, 27, 28, 29, 200, 4096, 4097):
        yield np.full(L, 121, np.uint8)
    dense = g.integers(0, 242, 5000).astype(np.uint8)       # no zero group at all (dense family)
    yield np.where(dense >= 121, dense + 1, dense).astype(np.uint8)
    for p in (0.1, 0.5, 0.9, 0.97, 0.995):
        for L in (1, 7, 8, 9, 100, 2047, 2048, 2049, 20000):
            yield np.where(g.random(L) < p, 121, g.integers(0, 243, L)).astype(np.uint8)
    # run lengths 1..100 and 14k-1/14k/14k+1 separated by literals
    menu = list(range(1, 101)) + [14 * k + d for k in range(1, 30) for d in (-1, 0, 1)]
    parts = []
    for r in menu:
        parts += [121] * r + [int(g.integers(0, 121))]
    yield np.array(parts, np.uint8)


@pytest.mark.parametrize("lane_mode", [0, 1, 2, 3, 4, 5])
@pytest.mark.parametrize("threads", [1, 2, 3, 8])
def test_scan_matches_oracle_zre(sim, threads, lane_mode):  # threads = warps per CTA
    """lane_mode 0: rows emitted from their kept literal lists; 1-3: the dense-row form,
    every lane's bytes emitted by lane_emit (variant 1, 2 or 3) into a 255-prefilled stage;
    4: variant 1 into the bank-padded stage (PadStage) K3 and K6c use; 5: variant 4 into it."""
    for i, B in enumerate(_streams()):
        ref = O.zre_encode(B)
        for nchunks in (1, 2, 3, 7, 64):
            got = sim(B, threads, nchunks, lane_mode)
            assert got.tolist() == ref.tolist(), (threads, nchunks, i, B.size, lane_mode)


def test_word_len_swar_matches_bytewise(sim):
    """K4 sums expansion lengths four bytes at a time (word_len): every byte value in
    every lane position, and random words, against the per-byte definition
    len(b) = b >= 243 ? b - 241 : 1 (inverse of P:545-546)."""
    import ctypes

    L = sim.lib
    L.tlc_word_len.restype = ctypes.c_uint32
    L.tlc_word_len.argtypes = [ctypes.c_uint32]

    def ref(w):
        return sum((b - 241 if b >= 243 else 1) for b in ((w >> (8 * i)) & 0xFF for i in range(4)))

    for b in range(256):
        for fill in (0, 121, 242, 243, 255):
            for pos in range(4):
                w = 0
                for i in range(4):
                    w |= (b if i == pos else fill) << (8 * i)
                assert L.tlc_word_len(w) == ref(w), (b, fill, pos)
    g = np.random.default_rng(5)
    for w in g.integers(0, 2**32, 20000, dtype=np.uint64):
        assert L.tlc_word_len(int(w)) == ref(int(w))
