"""Pins of the exchange oracle's aggregation (X3, reading R15) against things other than
itself: the hand-worked W = 2 / W = 3 steps of tests/golden/exchange_examples.json, and
an exact-rational replay of "average the gradients" -- the rank-ordered fold
of the dequantized pushes, each partial sum rounded to fp32 by an independent
round-to-nearest-even written here over Python Fractions, then the IEEE quotient by W --
at W = 2..8 on gradients whose scales differ per rank so that the fold's rounding is
visible.  The pushed trits are recovered from the payload bytes by a decoder written in
this file (ZRE expansion, base-3 digits), not by the oracle's decompress."""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import synth
from oracle import exchange as X

f32 = np.float32
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "exchange_examples.json")


@pytest.fixture(scope="module")
def ex():
    with open(GOLD) as f:
        return json.load(f)


def _h(x):
    return np.array([int(x, 16)], np.uint32).view(f32)[0]


def _bits(a):
    return np.asarray(a, f32).view(np.uint32).tolist()


def _run(case, grads):
    W, sizes, s = case["W"], case["sizes"], case["s"]
    ps = X.VirtualPS(sizes, W)
    assert [list(c) for c in ps.ctx] == case["plan"]
    outs = [[np.zeros(n, f32) for n in sizes] for _ in range(W)]
    means, sent = ps.push(grads, s)
    shared = ps.pull(means, outs, s)
    return ps, means, sent, shared, outs


def test_w2_hand_worked(ex):
    c = ex["w2"]
    grads = [[np.array(g, f32)] for g in c["grads"]]
    ps, means, sent, shared, outs = _run(c, grads)
    for r in range(2):
        for k in range(2):
            assert sent[r][k].payload.tolist() == c["push_payloads"][r][k]
            assert sent[r][k].M == f32(c["push_M"][r][k])
            assert _bits(ps.push_err[r][k]) == _bits(c["push_err"][r][k])
    for k in range(2):
        assert _bits(means[k]) == _bits(c["means"][k])
        assert shared[k].payload.tolist() == c["pull_payloads"][k]
        assert _bits(ps.pull_err[k]) == _bits(c["pull_err"][k])
    for r in range(2):
        assert _bits(outs[r][0]) == _bits(c["outs"])


def test_w3_hand_worked_rank_order_and_ieee_division(ex):
    c = ex["w3"]
    grads = [[np.array([_h(v) for v in g], f32)] for g in c["grads_hex"]]
    ps, means, sent, shared, outs = _run(c, grads)
    for r in range(3):
        for k in range(3):
            assert sent[r][k].payload.tolist() == c["push_payloads"][r][k], (r, k)
    for k in range(3):
        assert _bits(means[k]) == [int(v, 16) for v in c["means_hex"][k]], k
        assert shared[k].payload.tolist() == c["pull_payloads"][k]
        assert _bits(ps.pull_err[k]) == [int(v, 16) for v in c["pull_err_hex"][k]]
    assert _bits(ps.push_err[2][1]) == _bits(c["push_err_rank2_ctx1"])
    for r in range(3):
        assert _bits(outs[r][0]) == [int(v, 16) for v in c["outs_hex"]]
    # the pin is sharp: the exact mean and any other fold order give a different bit pattern
    exact = (Fraction(1) + 2 * Fraction(1, 2 ** 24)) / 3
    assert _bits([_round_f32(exact)])[0] == 0x3EAAAAAC != _bits(means[0])[0]


# ---------------------------------------------------------------- exact-rational replay
def _round_f32(x: Fraction) -> f32:
    """IEEE binary32 round-to-nearest-even of a rational (written out: no float
    arithmetic involved).  Returns +0 for 0; no overflow handling needed here."""
    if x == 0:
        return f32(0.0)
    neg = x < 0
    a = -x if neg else x
    e = a.numerator.bit_length() - a.denominator.bit_length()      # 2^e <= a < 2^(e+2)
    while Fraction(2) ** e > a:
        e -= 1
    while Fraction(2) ** (e + 1) <= a:
        e += 1
    e = max(e, -126)                                                  # subnormal spacing 2^-149
    ulp = Fraction(2) ** (e - 23)
    m = a / ulp
    lo = m.numerator // m.denominator
    rem = m - lo
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and lo % 2 == 1):
        lo += 1
    v = Fraction(lo) * ulp
    out = f32(float(v))                                               # v is exactly representable
    assert Fraction(float(out)) == v
    return f32(-out) if neg else out


def _decode_trits(payload, zre, n):
    """Payload bytes -> trits, from the paper's definitions: ZRE codes 243+(k-2) expand
    to k bytes of 121, byte j holds digits of elements j + i*P, digit =
    (B / 3^(4-i)) mod 3, trit = digit - 1."""
    B = []
    for b in payload.tolist():
        B.extend([121] * (b - 241) if zre and b >= 243 else [b])
    P = -(-n // 5)
    assert len(B) == P
    q = np.zeros(n, np.int64)
    for j in range(P):
        for i in range(5):
            e = i * P + j
            if e < n:
                q[e] = (B[j] // 3 ** (4 - i)) % 3 - 1
    return q


def _replay_mean(sent_c, n, W):
    acc = [Fraction(0)] * n
    qs = [_decode_trits(p.payload, True, n) for p in sent_c]
    for w in range(W):                                                # rank order (R15)
        Mw = Fraction(float(sent_c[w].M))
        for i in range(n):
            if qs[w][i] != 0:                                         # skip zero trits (R16)
                acc[i] = Fraction(float(_round_f32(acc[i] + Mw * int(qs[w][i]))))
    mean = np.array([_round_f32(a / W) for a in acc], f32)
    exact = [sum(Fraction(float(sent_c[w].M)) * int(qs[w][i]) for w in range(W)) / W for i in range(n)]
    bound = [(W + 1) * Fraction(1, 2 ** 24) * sum(Fraction(float(p.M)) for p in sent_c) / W] * n
    return mean, exact, bound


@pytest.mark.parametrize("W", [2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("s", [1.0, 1.9])
def test_mean_is_exact_rational_fold_then_ieee_division(W, s):
    sizes = [37, 211, 5]
    ps = X.VirtualPS(sizes, W)
    # per-rank scales 2^(3r) so that adding a later rank's M_w rounds the partial sum
    grads = [[(synth.gaussian(n, 97, r, t) * f32(2.0 ** (3 * r - 9))).astype(f32)
              for t, n in enumerate(sizes)] for r in range(W)]
    for step in range(2):
        if step:
            grads = [[(g * f32(-0.75)).astype(f32) for g in gr] for gr in grads]
        means, sent = ps.push(grads, s)
        for c, (t, lo, hi, _) in enumerate(ps.ctx):
            n = hi - lo
            mean, exact, bound = _replay_mean([sent[w][c] for w in range(W)], n, W)
            assert np.array_equal(mean.view(np.uint32), means[c].view(np.uint32)), (W, s, c)
            for i in range(n):
                assert abs(Fraction(float(means[c][i])) - exact[i]) <= bound[i]


def test_dropped_or_reordered_rank_is_detected():
    """Mutation check of the replay itself: a fold that skipped a rank or ran in reverse
    order does not reproduce the oracle's mean on these inputs."""
    W, sizes = 3, [60, 60, 60]                     # cap = 60: one whole-tensor context each
    ps = X.VirtualPS(sizes, W)
    # every trit nonzero: t = +-1 on rank 0 and +-2^-24 on ranks 1, 2, so the rank-ordered
    # partial sums hit ties (1 + 2^-24 -> 1) that a reverse fold avoids
    grads = [[(np.sign(synth.gaussian(60, 98, r, t)) * f32(1.0 if r == 0 else 2.0 ** -24)).astype(f32)
              for t in range(3)] for r in range(W)]
    means, sent = ps.push(grads, 1.0)
    n = ps.ctx[0][2] - ps.ctx[0][1]
    qs = [_decode_trits(sent[w][0].payload, True, n) for w in range(W)]
    Ms = [Fraction(float(sent[w][0].M)) for w in range(W)]

    def fold(order):
        out = []
        for i in range(n):
            a = Fraction(0)
            for w in order:
                if qs[w][i]:
                    a = Fraction(float(_round_f32(a + Ms[w] * int(qs[w][i]))))
            out.append(_round_f32(a / W))
        return np.array(out, f32).view(np.uint32)

    assert np.array_equal(fold([0, 1, 2]), means[0].view(np.uint32))
    assert not np.array_equal(fold([2, 1, 0]), means[0].view(np.uint32))
    assert not np.array_equal(fold([0, 1]), means[0].view(np.uint32))


def test_round_f32_against_numpy_on_float64_exact_values():
    rng = np.random.default_rng(5)
    for x in rng.standard_normal(2000) * 10.0 ** rng.integers(-40, 38, 2000):
        # float64 -> float32 is a single correct rounding when x itself is the exact value
        assert _round_f32(Fraction(float(x))).view(np.uint32) == f32(x).view(np.uint32)
    assert _round_f32(Fraction(1) + Fraction(1, 2 ** 24)) == f32(1.0)                # tie -> even
    assert _round_f32(Fraction(1) + Fraction(3, 2 ** 24)) == f32(1.0 + 2 ** -22)       # tie -> even (up)
    assert _round_f32(Fraction(1, 2 ** 149)).view(np.uint32) == 1                      # smallest subnormal


def test_failed_push_poisons_only_its_context():
    """Reading R24: a NaN in one rank's push gives that context a NaN mean (an fp32 sum
    with a NaN term is NaN), its shared pull fails with NONFINITE and is applied nowhere;
    every other context is exactly what it is without the failure."""
    W, sizes = 3, [40, 40, 40]
    grads = [[synth.gaussian(40, 99, r, t) for t in range(3)] for r in range(W)]
    ref = X.VirtualPS(sizes, W)
    ref_means, _ = ref.push(grads, 1.5)
    bad = [[g.copy() for g in gr] for gr in grads]
    bad[1][2][5] = np.nan
    ps = X.VirtualPS(sizes, W)
    means, sent = ps.push(bad, 1.5)
    c_bad = [c for c, (t, _, _, _) in enumerate(ps.ctx) if t == 2][0]
    assert sent[1][c_bad].status == 2                                  # NONFINITE (R6)
    assert np.array_equal(ps.push_err[1][c_bad], np.zeros(40, f32))     # err untouched (R6)
    for c in range(len(ps.ctx)):
        if c == c_bad:
            assert np.isnan(means[c]).all()
        else:
            assert np.array_equal(means[c].view(np.uint32), ref_means[c].view(np.uint32))
    outs = [[np.zeros(40, f32) for _ in sizes] for _ in range(W)]
    shared = ps.pull(means, outs, 1.5)
    assert shared[c_bad].status == 2
    assert np.array_equal(ps.pull_err[c_bad], np.zeros(40, f32))
    for r in range(W):
        assert np.array_equal(outs[r][2], np.zeros(40, f32))
        assert not np.array_equal(outs[r][0], np.zeros(40, f32))
