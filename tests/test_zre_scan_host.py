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


def test_producer_seek_entries_match_payload_scan(sim):
    """The seek entries K3 writes for the peer-memory consumers (exchange): K3's decomposition
    as built (chunks of 8 or 32 KiB, warps on whole 1 KiB rows), recording (payload offset << 4)
    | run carry at every row start that is a multiple of 4096.  K5 needs a byte index i and a
    skip with start(i) + skip = J0 and skip <= len(i), len(b) = b >= 243 ? b - 241 : 1 (inverse
    of P:545-546), start walked here over the oracle's encoding byte by byte.  K4's entry is the
    byte covering J0; K3's equals it except where J0 holds a literal after c > 0 pending zero
    groups: then it names the flush code of those c groups (emitted next) with skip = c, its
    whole expansion (DESIGN reading R25) -- checked to be exactly that case."""
    L = sim.lib
    L.zre_seek_sim.restype = ctypes.c_uint64
    L.zre_seek_sim.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint64,
                               ctypes.c_void_p, ctypes.c_void_p]
    g = synth.rng(73)
    cases = []
    for p in (0.0, 0.5, 0.9, 0.99, 1.0):
        for n in (4096, 4097, 3 * 8192 + 4096 + 37, 2 * 32768 + 5 * 4096 + 100, 5 * 32768 + 11):
            cases.append(np.where(g.random(n) < p, 121, g.integers(0, 243, n)).astype(np.uint8))
    runs = []                                          # runs straddling tile starts at every carry
    for r in list(range(1, 30)) + [4095, 4096, 4097, 14 * 300 + 3]:
        runs += [121] * r + [int(g.integers(0, 121))]
    cases.append(np.array(runs, np.uint8))
    alt = 0
    for B in cases:
        ref = O.zre_encode(B)
        lens = np.where(ref >= 243, ref.astype(np.int64) - 241, 1)
        start = np.concatenate([[0], np.cumsum(lens)[:-1]])
        assert int(lens.sum()) == B.size
        ntiles = -(-B.size // 4096)
        want = []
        for k in range(ntiles):
            i = int(np.searchsorted(start, 4096 * k, side="right")) - 1
            want.append((i << 4) | (4096 * k - int(start[i])))
        for chunk in (8192, 32768):
            out = np.full(B.size + 16, 0xEE, np.uint8)
            seek = np.full(ntiles, 0xFFFFFFFFFFFFFFFF, np.uint64)
            z = L.zre_seek_sim(B.ctypes.data, B.size, 8, chunk, out.ctypes.data, seek.ctypes.data)
            assert out[:z].tolist() == ref.tolist(), (B.size, chunk)
            for k, (got, w) in enumerate(zip(seek.tolist(), want)):
                i, skip = got >> 4, got & 15
                assert int(start[i]) + skip == 4096 * k and skip <= int(lens[i]), (B.size, chunk, k)
                if got != w:                       # a fully skipped flush code before J0's literal
                    assert skip == int(lens[i]) and (w >> 4) == i + 1 and (w & 15) == 0, (B.size, chunk, k)
                    assert B[4096 * k] != 121 and B[4096 * k - 1] == 121, (B.size, chunk, k)
                    alt += 1
    assert alt > 0                                  # the flush-code form was exercised
