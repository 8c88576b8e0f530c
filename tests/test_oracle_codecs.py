"""Pins of the oracle's compared-design codecs (Sec. 5.1):
"Stoch 3-value + QE" and "8-bit int".

Pinned against: the Random123 known-answer vectors of Philox4x32-10
(tests/golden/philox_kat.json), triton's own Philox (an independent library
implementation, run in its CPU interpreter), SPEC's worked examples,
exact rational arithmetic, and the statistical property that defines stochastic
quantization ("expectation matches their input value").
"""
import json
import math
import os
import subprocess
import sys
from fractions import Fraction

import numpy as np
import pytest

import oracle as O

f32 = np.float32
HERE = os.path.dirname(os.path.abspath(__file__))


# --------------------------------------------------------------------------- Philox
def test_philox_known_answers():
    with open(os.path.join(HERE, "golden", "philox_kat.json")) as f:
        kat = json.load(f)["philox4x32_10"]
    for v in kat:
        ctr = [int(x, 16) for x in v["ctr"]]
        key = [int(x, 16) for x in v["key"]]
        assert [int(x) for x in O.philox4x32_10(ctr, key)] == [int(x, 16) for x in v["out"]]


_TRITON = r"""
import os, sys, json
os.environ["TRITON_INTERPRET"] = "1"
import torch, triton, triton.language as tl

@triton.jit
def k(out, seed, N: tl.constexpr):
    off = tl.arange(0, N)
    a, b, c, d = tl.randint4x(seed, off, n_rounds=10)
    tl.store(out + off * 4 + 0, a)
    tl.store(out + off * 4 + 1, b)
    tl.store(out + off * 4 + 2, c)
    tl.store(out + off * 4 + 3, d)

res = {}
for seed in (0x12345678ABCDEF, 7, 0xFFFFFFFF00000001):
    o = torch.zeros(64 * 4, dtype=torch.int32)
    k[(1,)](o, seed, 64)
    res[str(seed)] = [x & 0xFFFFFFFF for x in o.tolist()]
print(json.dumps(res))
"""


def test_philox_matches_triton():
    """triton.language.randint4x(seed, offset) = Philox4x32-10 at counter (offset, 0, 0, 0)
    under key (seed low, seed high): a second, independent implementation."""
    r = subprocess.run([sys.executable, "-c", _TRITON], capture_output=True, text=True, timeout=600)
    if r.returncode != 0:
        pytest.skip("triton interpreter unavailable: " + r.stderr[-300:])
    res = json.loads(r.stdout.strip().splitlines()[-1])
    for seed, words in res.items():
        seed = int(seed)
        key = [seed & 0xFFFFFFFF, seed >> 32]
        for off in range(64):
            assert [int(x) for x in O.philox4x32_10([off, 0, 0, 0], key)] == words[4 * off: 4 * off + 4]


def test_stoch_word_counter_layout():
    """R22: element e takes word e%4 of the block at counter (e/4 lo, e/4 hi, step lo, step hi)."""
    seed, step = 0x0123456789ABCDEF, (5 << 32) | 9
    key = [seed & 0xFFFFFFFF, seed >> 32]
    for e in [0, 1, 2, 3, 4, 7, 8, 1001, (1 << 34) + 6]:
        b = e // 4
        blk = O.philox4x32_10([b & 0xFFFFFFFF, b >> 32, step & 0xFFFFFFFF, step >> 32], key)
        assert O.stoch_word(seed, step, e) == int(blk[e % 4])


# --------------------------------------------------------------------------- stochastic 3-value
def test_stoch_boundaries():
    """x = m is always sign(x); x = 0 is always 0; m = 0 gives zeros."""
    t = np.array([1.0, -1.0, 0.0, -0.0, 0.25], dtype=f32)
    for step in range(200):
        st, m, q = O.stoch_quantize(t, 11, step)
        assert st == O.OK and m == f32(1.0)
        assert q[0] == 1 and q[1] == -1 and q[2] == 0 and q[3] == 0 and q[4] in (0, 1)
    st, m, q = O.stoch_quantize(np.zeros(9, dtype=f32), 3, 0)
    assert st == O.OK and m == 0 and not q.any()
    for bad in (np.nan, np.inf, -np.inf):
        st, _, _ = O.stoch_quantize(np.array([0.5, bad], dtype=f32), 1, 0)
        assert st == O.ERR_NONFINITE


def test_stoch_half_uses_top_bit():
    """|x|/m = 1/2 exactly: U = (w >> 8)/2^24 < 1/2 iff bit 31 of w is 0 -- pins which bits
    make U (a mask of the low 24 bits would decide on bit 23 instead)."""
    n = 4096
    t = np.full(n, 0.5, dtype=f32)
    t[0] = 1.0
    t[1::3] = -0.5
    seed, step = 99, 3
    st, m, q = O.stoch_quantize(t, seed, step)
    key = [seed, 0]
    for e in range(1, n):
        b = e // 4
        w = int(O.philox4x32_10([b, 0, step, 0], key)[e % 4])
        expect = 0 if (w >> 31) else (1 if t[e] > 0 else -1)
        assert q[e] == expect, e


def test_stoch_decision_exact_rational():
    """q = sign(x) iff U < fl(|x|/m) with U = (w>>8)/2^24: checked with exact rationals on
    random values, the quotient rounded by numpy's IEEE float32 division."""
    rng = np.random.default_rng(5)
    t = rng.standard_normal(3000).astype(f32)
    seed, step = 1234567, 42
    st, m, q = O.stoch_quantize(t, seed, step)
    assert m == np.abs(t).max()
    for e in range(t.size):
        w = O.stoch_word(seed, step, e)
        U = Fraction(w >> 8, 1 << 24)
        p = Fraction(float(np.abs(t[e]) / m))          # IEEE fp32 quotient
        expect = (1 if t[e] > 0 else -1) if U < p else 0
        assert q[e] == expect


def test_stoch_unbiased():
    """E[m*q] = x.  20,000 independent steps per element; the mean of m*q is
    within 4.5 standard errors of x (binomial: sd = m*sqrt(p(1-p)/K))."""
    t = np.array([1.0, 0.3, -0.7, 0.05, -0.5, 0.0, 0.999, -0.01], dtype=f32)
    K = 20000
    acc = np.zeros(t.size)
    for step in range(K):
        st, m, q = O.stoch_quantize(t, 77, step)
        acc += q
    mean = acc / K
    for x, mu in zip(t.astype(float), mean):
        p = abs(x)
        se = math.sqrt(p * (1 - p) / K) + 1e-12
        assert abs(mu - x) <= 4.5 * se + 1e-9, (x, mu)


def test_stoch_compress_is_qe_of_trits():
    """The payload is the quartic (+ZRE) encoding of the stochastic trits, decodable by the
    3LC decompressor with M = m ("our quartic encoding")."""
    rng = np.random.default_rng(8)
    for n in [1, 5, 7, 1000, 4099]:
        t = rng.standard_normal(n).astype(f32)
        st, m, q = O.stoch_quantize(t, 5, n)
        for zre in (False, True):
            c = O.stoch_compress(t, 5, n, zre)
            assert c.status == O.OK and c.M == m
            B = O.quartic_encode(q)
            assert np.array_equal(c.payload, O.zre_encode(B) if zre else B)
            st2, out = O.decompress(c.payload, zre, c.M, n)
            assert st2 == O.OK
            assert np.array_equal(out, (m * q.astype(f32)).astype(f32))
            if not zre:
                assert c.payload_len == -(-n // 5)      # 1.6 bits per value


def test_stoch_seed_and_step_change_draws():
    t = np.full(1000, 0.5, dtype=f32)
    t[0] = 1.0
    a = O.stoch_quantize(t, 1, 0)[2]
    assert np.array_equal(a, O.stoch_quantize(t, 1, 0)[2])          # determinism
    assert not np.array_equal(a, O.stoch_quantize(t, 2, 0)[2])
    assert not np.array_equal(a, O.stoch_quantize(t, 1, 1)[2])


# --------------------------------------------------------------------------- 8-bit int
def test_int8_spec_examples():
    st, sc, c = O.int8_compress(np.array([1.27, -1.27], dtype=f32))
    assert st == O.OK and sc == f32(1.27) / f32(127) and c.tolist() == [127, -127]
    assert abs(float(sc) - 0.01) < 1e-9
    st, sc, c = O.int8_compress(np.zeros(2, dtype=f32))
    assert st == O.OK and sc == 0 and c.tolist() == [0, 0]


def test_int8_ties_round_away():
    """scale = 1 (max 127): 2.5 -> 3 and -2.5 -> -3 (half away, R1; half-even gives 2)."""
    t = np.array([127.0, 2.5, -2.5, 0.5, -0.5, 1.5, 126.5, -0.49999997], dtype=f32)
    st, sc, c = O.int8_compress(t)
    assert sc == 1.0 and c.tolist() == [127, 3, -3, 1, -1, 2, 127, 0]


def test_int8_exact_rational_and_bounds():
    """codes = the integer nearest fl(t/scale) (ties away) -- exact rationals over numpy's
    IEEE quotient; codes in [-127,127] (P:626 '-128 unused'); |t - scale*code| <= scale/2
    up to the quotient's rounding."""
    rng = np.random.default_rng(9)
    for scale_t in [1.0, 1e-30, 3e20]:
        t = (rng.standard_normal(5000) * scale_t).astype(f32)
        st, sc, c = O.int8_compress(t)
        assert sc == np.abs(t).max() / f32(127)
        assert c.min() >= -127 and c.max() <= 127
        for x, k in zip(t, c):
            v = Fraction(float(x / sc))
            r = math.floor(abs(v) + Fraction(1, 2)) * (1 if v >= 0 else -1)
            r = max(-127, min(127, r))
            assert k == r
        out = O.int8_decompress(c, sc)
        assert np.array_equal(out, (sc * c.astype(f32)).astype(f32))
        assert np.all(np.abs(t.astype(np.float64) - out) <= float(sc) * (0.5 + 1e-6))


def test_int8_accumulate_and_errors():
    t = np.array([1.0, 0.001, -0.5, 0.0], dtype=f32)
    st, sc, c = O.int8_compress(t)
    base = np.array([10.0, -0.0, 2.0, -0.0], dtype=f32)
    out = O.int8_decompress(c, sc, base.copy(), accumulate=True)
    assert c[1] == 0 and c[3] == 0
    assert out[1].tobytes() == f32(-0.0).tobytes()                 # code 0: untouched (R16)
    assert out[0] == f32(10.0) + sc * f32(c[0])
    st, _, _ = O.int8_compress(np.array([1.0, np.nan], dtype=f32))
    assert st == O.ERR_NONFINITE
    st, sc, c = O.int8_compress(np.array([1e-45, -1e-45], dtype=f32))   # scale underflows (R23)
    assert st == O.OK and sc == 0 and not c.any()
