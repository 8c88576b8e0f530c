"""Pins of the CPU oracle (oracle/tlc_oracle.c) against things other than itself.

Every test checks the oracle against what PAPER.md / SPEC.md print (tests/golden),
closed forms, invariants the mathematics fixes, a textbook routine, or brute force
against an independently written second implementation.  Chosen so that a dropped
term, wrong sign/index, transposed partition or wrong rounding mode fails one.
"""
import itertools
import math
import struct

import numpy as np
import pytest

import oracle as O
import synth

f32 = np.float32


# --------------------------------------------------------------------------- golden values
def test_golden_quantize(golden):
    for ex in golden["quantize"]:
        t = np.array(ex["t"], dtype=f32)
        st, M, a = O.scale(t, ex["s"])
        assert st == O.OK
        if "M" in ex:
            assert M == f32(ex["M"]), ex["cite"]
        else:
            assert M == f32(ex["M_f32_product"][0]) * f32(ex["M_f32_product"][1])
        assert O.quantize(t, M).tolist() == ex["q"], ex["cite"]


def test_golden_dequantize(golden):
    for ex in golden["dequantize"]:
        out = O.dequantize(np.array(ex["q"], dtype=np.int8), f32(ex["M"]))
        assert out.tolist() == np.array(ex["out"], dtype=f32).tolist(), ex["cite"]


def test_golden_context_compress(golden):
    for ex in golden["context_compress"]:
        buf = np.array(ex["buffer"], dtype=f32)
        c = O.compress(np.array(ex["t"], dtype=f32), buf, ex["s"], use_zre=False)
        assert c.status == O.OK
        assert c.M == f32(ex["M"])
        st, q = O.quartic_decode(c.payload, len(ex["t"]))
        assert q.tolist() == ex["q"], ex["cite"]
        assert buf.tolist() == np.array(ex["new_buffer"], dtype=f32).tolist(), ex["cite"]


def test_golden_quartic(golden):
    for ex in golden["quartic"]:
        B = O.quartic_encode(np.array(ex["q"], dtype=np.int8))
        assert B.tolist() == ex["bytes"], ex["cite"]
        st, q = O.quartic_decode(B, len(ex["q"]))
        assert st == O.OK and q.tolist() == ex["q"]


def test_golden_zre(golden):
    for ex in golden["zre"]:
        Z = O.zre_encode(np.array(ex["bytes"], dtype=np.uint8))
        assert Z.tolist() == ex["zre"], ex["cite"]
        st, B = O.zre_decode(Z, len(ex["bytes"]))
        assert st == O.OK and B.tolist() == ex["bytes"]


def test_golden_pipeline(golden):
    for ex in golden["pipeline"]:
        t = np.zeros(ex["zeros"], dtype=f32) if "zeros" in ex else np.array(ex["t"], dtype=f32)
        buf = np.zeros_like(t)
        c = O.compress(t, buf, ex["s"], ex["use_zre"])
        assert c.status == O.OK and c.M == f32(ex["M"])
        if "payload" in ex:
            assert c.payload.tolist() == ex["payload"], ex["cite"]
        if "payload_len" in ex:
            assert c.payload_len == ex["payload_len"], ex["cite"]
            assert c.payload[-len(ex["payload_tail"]):].tolist() == ex["payload_tail"]


def test_golden_decompress(golden):
    for ex in golden["decompress"]:
        st, out = O.decompress(np.array(ex["payload"], dtype=np.uint8), ex["use_zre"], f32(ex["M"]), ex["n"])
        assert st == O.OK
        assert out.tolist() == np.array(ex["out"], dtype=f32).tolist(), ex["cite"]


def test_golden_ratios(golden):
    r = golden["ratio"]
    # 280x for the all-zero fp32 tensor: 70 zeros -> 1 payload byte.
    c = O.compress(np.zeros(r[0]["zeros"], f32), np.zeros(r[0]["zeros"], f32), 1.0, True)
    assert 4 * c.n / c.payload_len == r[0]["ratio"]
    # Table 2 "No ZRE" 20.0x / 1.60 bits for n a multiple of 5, any data.
    for n in (5, 500, 12345):
        t = synth.gaussian(n, 7, n)
        c = O.compress(t, np.zeros(n, f32), 1.0, False)
        assert 4 * n / c.payload_len == r[1]["ratio_no_zre"]
        assert 8 * c.payload_len / n == r[1]["bits_no_zre"]
    # 1.6 bits is 0.95% over log2(3); 2 bits is ~26% over.
    assert round(100 * (r[2]["bits"] / math.log2(3) - 1), 2) == r[2]["overhead_pct"]
    assert round(100 * (r[3]["bits"] / math.log2(3) - 1)) == r[3]["overhead_pct"]


def test_all_zero_280x_many_sizes():
    # P:546-548 / S:245: 70*r zeros -> exactly r bytes of 255.
    for r in (1, 2, 3, 17, 1000):
        n = 70 * r
        c = O.compress(np.zeros(n, f32), np.zeros(n, f32), 1.9, True)
        assert c.payload.tolist() == [255] * r
        assert 4 * n / c.payload_len == 280.0


# --------------------------------------------------------------------------- brute force
def test_quartic_bijection_all_243_groups():
    """3^5 = 243 trit groups; step 6 is the base-3 number p0p1p2p3p4,
    checked against Python's int(str, 3) (a textbook base conversion)."""
    seen = set()
    for trits in itertools.product((-1, 0, 1), repeat=5):
        B = O.quartic_encode(np.array(trits, dtype=np.int8))
        expect = int("".join(str(t + 1) for t in trits), 3)
        assert B.tolist() == [expect]
        seen.add(int(B[0]))
        st, q = O.quartic_decode(B, 5)
        assert st == O.OK and tuple(q.tolist()) == trits
    assert seen == set(range(243))


def test_quartic_partition_layout_random():
    """P:508-509 'Divide the array into 5 partitions': byte j holds elements
    j, j+P, ..., j+4P (R9).  Checked via Python int(str, 3) per byte."""
    g = synth.rng(11)
    for n in list(range(1, 41)) + [97, 1000, 4099]:
        q = g.integers(-1, 2, size=n).astype(np.int8)
        B = O.quartic_encode(q)
        P = -(-n // 5)
        assert B.size == P
        padded = list(q + 1) + [0] * (5 * P - n)
        for j in range(P):
            digits = "".join(str(int(padded[k * P + j])) for k in range(5))
            assert int(B[j]) == int(digits, 3)
        st, back = O.quartic_decode(B, n)
        assert st == O.OK and np.array_equal(back, q)


def _naive_zre(bs):
    """Second, independent ZRE: groupby runs, divmod into 14-chunks."""
    out = []
    for v, grp in itertools.groupby(bs):
        k = len(list(grp))
        if v != 121:
            out += [v] * k
            continue
        full, rem = divmod(k, 14)
        out += [255] * full
        if rem == 1:
            out.append(121)
        elif rem >= 2:
            out.append(243 + rem - 2)
    return out


def test_zre_all_binary_patterns_up_to_16():
    for L in range(0, 17):
        for bits in itertools.product((0, 1), repeat=L):
            bs = [121 if b else 7 for b in bits]
            Z = O.zre_encode(np.array(bs, dtype=np.uint8)).tolist()
            assert Z == _naive_zre(bs)
            assert len(Z) <= len(bs)                         # never expands
            assert all(not (a == 121 and b == 121) for a, b in zip(Z, Z[1:]))  # canonical
            st, back = O.zre_decode(np.array(Z, dtype=np.uint8), len(bs))
            assert st == O.OK and back.tolist() == bs


def test_zre_runs_1_to_200_and_random():
    g = synth.rng(12)
    for k in range(1, 201):
        bs = [3] + [121] * k + [242]
        assert O.zre_encode(np.array(bs, dtype=np.uint8)).tolist() == _naive_zre(bs)
    for _ in range(200):
        L = int(g.integers(1, 3000))
        bs = np.where(g.random(L) < 0.9, 121, g.integers(0, 243, size=L)).astype(np.uint8)
        Z = O.zre_encode(bs)
        assert Z.tolist() == _naive_zre(bs.tolist())
        st, back = O.zre_decode(Z, L)
        assert st == O.OK and np.array_equal(back, bs)


def test_zre_decode_rejects_malformed():
    # expansion length must equal the declared length.
    assert O.zre_decode(np.array([255], np.uint8), 13)[0] == O.ERR_FORMAT   # overrun
    assert O.zre_decode(np.array([255], np.uint8), 15)[0] == O.ERR_FORMAT   # short
    assert O.zre_decode(np.array([], np.uint8), 1)[0] == O.ERR_FORMAT
    assert O.quartic_decode(np.array([243], np.uint8), 5)[0] == O.ERR_FORMAT  # > 242
    st, _ = O.decompress(np.array([121, 121], np.uint8), False, f32(1), 5)   # len != P
    assert st == O.ERR_FORMAT


def test_all_zero_closed_form():
    """Pads are digit 0 (R10) at the last k = 5P - n bytes (byte 120); the other
    P - k bytes are 121 -> Z = ceil((P-k)/14) + k for P >= 4."""
    for n in range(16, 3000):
        P = -(-n // 5)
        k = 5 * P - n
        c = O.compress(np.zeros(n, f32), np.zeros(n, f32), 1.0, True)
        assert c.payload_len == -(-(P - k) // 14) + k
        assert c.payload[c.payload_len - k:].tolist() == [120] * k


# --------------------------------------------------------------------------- quantization
def _next_down(x):
    return np.nextafter(f32(x), f32(-np.inf), dtype=f32)


def test_round_half_away_ties():
    """Eq. 2 with round half away from zero (R1): u = +-M/2 exactly -> +-1,
    the float just inside -> 0."""
    for M in (f32(1.0), f32(0.4), f32(3.5), f32(1e-30), f32(6.0e37)):
        half = M / f32(2)
        u = np.array([half, -half, _next_down(half), -_next_down(half), M, -M, 0.0], dtype=f32)
        assert O.quantize(u, M).tolist() == [1, -1, 0, 0, 1, -1, 0]


def test_quantize_matches_exact_rational_rounding():
    """Independent check of Eq. 2 in exact rationals: fl32(u/M) >= 1/2 iff
    |u/M| >= 1/2 - 2^-26 (the midpoint between 1/2 and its fp32 predecessor
    1/2 - 2^-25; the tie rounds to the even 1/2), then half away from zero."""
    from fractions import Fraction

    g = synth.rng(13)
    thr = Fraction(1, 2) - Fraction(1, 2 ** 26)
    checked = 0
    for _ in range(4000):
        M = f32(np.exp(g.uniform(-80, 80)))
        near = g.random() < 0.5
        x = f32(0.5) + f32(g.integers(-3, 4)) * f32(2.0 ** -25) if near else f32(g.uniform(-1, 1))
        u = f32(x * M) * (f32(-1) if g.random() < 0.5 else f32(1))
        if not np.isfinite(u) or M == 0 or abs(u) > M:
            continue
        r = Fraction(float(u)) / Fraction(float(M))
        expect = (1 if r > 0 else -1) if abs(r) >= thr else 0
        assert int(O.quantize(np.array([u], f32), M)[0]) == expect, (u, M)
        checked += 1
    assert checked > 3000


def test_error_bound_and_conservation():
    """|T_in - T_out| <= M/2 and M/2 < max|T_in| for 1 <= s < 2;
    steps (a),(b): buffer + M*q == u exactly (Sterbenz: M/2 <= |u| <= M when q != 0)."""
    g = synth.rng(14)
    for s in (1.0, 1.5, 1.75, 1.9, 1.9999999):
        for dist in ("normal", "laplace", "t3"):
            n = 20000
            if dist == "normal":
                t = g.standard_normal(n).astype(f32)
            elif dist == "laplace":
                t = g.laplace(size=n).astype(f32)
            else:
                t = g.standard_t(3, size=n).astype(f32)
            buf = (0.1 * g.standard_normal(n)).astype(f32)
            u = (buf + t).astype(f32)
            c = O.compress(t, buf, s, use_zre=True)
            st, out = O.decompress(c.payload, True, c.M, n)
            assert st == O.OK
            a = np.max(np.abs(u))
            assert c.M == a * f32(s)
            d = np.abs(u.astype(np.float64) - out.astype(np.float64))
            assert np.all(d <= float(c.M) / 2)
            assert float(c.M) / 2 < float(a)
            assert np.array_equal(buf, u - out)                     # residual is the error
            assert np.array_equal((buf + out).view(np.uint32), u.view(np.uint32)) or \
                np.array_equal(buf + out, u)                         # exact conservation


def test_signed_zero_residual():
    """R8: zero trit -> u - (+0): a -0 input keeps -0 in the buffer."""
    t = np.array([-0.0, 0.0, 1.0, -0.0], dtype=f32)
    buf = np.array([-0.0, -0.0, 0.0, 0.0], dtype=f32)
    c = O.compress(t, buf, 1.0, True)
    assert c.status == O.OK
    assert [math.copysign(1, x) for x in buf.tolist()] == [-1, 1, 1, 1]


def test_zero_count_monotone_in_s():
    """S:150 / P:387-392: a larger s gives a sparser quantized tensor."""
    g = synth.rng(15)
    for trial in range(20):
        t = g.standard_normal(5000).astype(f32)
        zs = []
        for s in (1.0, 1.25, 1.5, 1.75, 1.9):
            st, M, _ = O.scale(t, s)
            zs.append(int(np.sum(O.quantize(t, M) == 0)))
        assert zs == sorted(zs)


def test_max_element_quantizes_exactly_with_s1():
    """s = 1: M = max|u|, so the arg-max element maps to +-1 with zero residual."""
    g = synth.rng(16)
    t = g.standard_normal(999).astype(f32)
    buf = np.zeros_like(t)
    i = int(np.argmax(np.abs(t)))
    c = O.compress(t, buf, 1.0, True)
    assert buf[i] == 0.0 and c.M == abs(t[i])


def test_roundtrip_is_dequantized_quantization():
    """decompress(compress(u)) == M * round(u/M) exactly (QE + ZRE lossless)."""
    g = synth.rng(17)
    for n in list(range(1, 60)) + [1000, 4097, 65536]:
        for fam in ("gauss", "runs"):
            t = synth.gaussian(n, 17, n) if fam == "gauss" else synth.runs_adversarial(n, 1.0, 17, n)
            buf = (0.5 * g.standard_normal(n)).astype(f32)
            u = O.accumulate(t, buf)
            for s in (1.0, 1.75):
                b2 = buf.copy()
                c = O.compress(t, b2, s, True)
                st, out = O.decompress(c.payload, True, c.M, n)
                assert st == O.OK
                st2, M, _ = O.scale(u, s)
                assert M == c.M
                assert np.array_equal(out, O.dequantize(O.quantize(u, M), M))


def test_nonfinite_and_range_leave_buffer_untouched():
    """S:33/S:70 (R6): NaN/Inf -> NONFINITE; max*s overflow -> RANGE; buffer unchanged."""
    for bad, code, s in ((np.nan, O.ERR_NONFINITE, 1.0), (np.inf, O.ERR_NONFINITE, 1.0),
                         (-np.inf, O.ERR_NONFINITE, 1.0),
                         (np.finfo(f32).max, O.ERR_RANGE, 1.5)):
        for pos in (0, 5, 9):
            t = np.ones(10, f32)
            t[pos] = bad
            buf = np.arange(10, dtype=f32) * f32(0.01)
            ref = buf.copy()
            c = O.compress(t, buf, s, True)
            assert c.status == code
            assert np.array_equal(buf, ref)
    # FLT_MAX with s = 1 is representable -> OK
    t = np.array([np.finfo(f32).max, 1.0], f32)
    assert O.compress(t, np.zeros(2, f32), 1.0, True).status == O.OK


def test_argument_errors():
    """s outside [1, 2) is a hard error."""
    for s in (0.999, 2.0, -1.0, float("nan")):
        assert O.compress(np.ones(3, f32), np.zeros(3, f32), s, True).status == O.ERR_ARG


def test_telescoping_conservation_multistep():
    """sum of decompressed outputs + final buffer == sum of inputs (up to
    the fp32 rounding of the accumulate step)."""
    n = 4000
    buf = np.zeros(n, f32)
    tot_in = np.zeros(n, np.float64)
    tot_out = np.zeros(n, np.float64)
    for step in range(30):
        t = synth.gaussian(n, 18, step)
        tot_in += t
        c = O.compress(t, buf, 1.75, True)
        st, out = O.decompress(c.payload, True, c.M, n)
        tot_out += out
    err = np.abs(tot_out + buf - tot_in)
    assert np.max(err) <= 1e-5 * max(1.0, np.max(np.abs(tot_in))) * 30


def test_accumulate_mode_skips_zero_trits():
    """R16: ACCUMULATE adds M*q only where q != 0 (a -0 target stays -0)."""
    out = np.array([-0.0, 1.0, 2.0, -0.0, 5.0], f32)
    st, res = O.decompress(np.array([175], np.uint8), True, f32(0.5), 5, out=out.copy(), accumulate=True)
    # q = [1, -1, 0, 0, 0]
    assert st == O.OK
    assert res.tolist() == [0.5, 0.5, 2.0, -0.0, 5.0]
    assert math.copysign(1, res[3]) == -1


def test_determinism():
    t = synth.gaussian(10007, 19)
    a, b = np.zeros_like(t), np.zeros_like(t)
    ca, cb = O.compress(t, a, 1.5, True), O.compress(t, b, 1.5, True)
    assert np.array_equal(ca.payload, cb.payload) and np.array_equal(a, b)


def test_s_is_fp32():
    """R3: s is an fp32 (1.9f = 1.89999997615814208984375)."""
    t = np.array([1.0], f32)
    st, M, _ = O.scale(t, 1.9)
    assert struct.pack("<f", M) == struct.pack("<f", 1.9)
    assert float(M) == 1.89999997615814208984375


def test_malformed_scale_is_format():
    """R21: Eq. 1 gives a finite M >= +0; a header with M < 0, -0, NaN or Inf is malformed."""
    for M in (-1.0, -0.0, float("nan"), float("inf")):
        st, _ = O.decompress(np.array([175], np.uint8), True, f32(M), 5)
        assert st == O.ERR_FORMAT


def test_openmp_build_is_bitwise_identical():
    """bench.py's cpu_baseline times the -fopenmp build of the same oracle source; it must
    compute exactly what the plain build computes (independent element-wise loops, exact
    max), including the NONFINITE decision and the untouched buffer."""
    import synth

    results = []
    for omp in (False, True):
        O.use_openmp(omp)
        try:
            r = []
            for n, s in ((1, 1.0), (1000, 1.9), (300_007, 1.75)):
                t = synth.gaussian(n, 77, n)
                buf = (0.5 * synth.gaussian(n, 78, n)).astype(np.float32)
                c = O.compress(t, buf, s)
                st, out = O.decompress(c.payload, True, c.M, n)
                acc = buf.copy()
                st2, acc = O.decompress(c.payload, True, c.M, n, out=acc, accumulate=True)
                bad = t.copy()
                bad[n // 2] = np.nan
                b2 = buf.copy()
                cb = O.compress(bad, b2, s)
                r.append((c.payload.tobytes(), float(c.M), buf.tobytes(), out.tobytes(), acc.tobytes(), st, st2,
                          cb.status, b2.tobytes()))
            results.append(r)
        finally:
            O.use_openmp(False)
    assert results[0] == results[1]
