"""Eq. 2 on the GPU (compare form for M >= 2^-125, IEEE quotient below, DESIGN.md
5.2) against the oracle's roundf(u / M), float by float.

For each scale regime the input holds the maximum a (so M = fl(a*s)) and every
fp32 value in bands around the decision points M/2 and M (2^16 consecutive
floats on each side, both signs), plus random values.  The quartic bytes (no
ZRE) and the error buffer must match bit for bit.  TLC_EXHAUSTIVE=1 extends the
sweep to every float with |u| <= a for a = 1 (about 2.1e9 values)."""
import os

import numpy as np
import pytest

import oracle as O
import synth

pytestmark = pytest.mark.gpu
f32 = np.float32

REGIMES = [  # (a = max|u|, s)
    (f32(1.0), 1.0), (f32(1.0), 1.9), (f32(3.0), 1.5), (f32(1e-30), 1.75),
    (f32(2.0 ** -124), 1.0),        # M = 2^-124: compare form, M/2 normal
    (f32(2.0 ** -125), 1.0),        # M = 2^-125: the boundary of the compare form
    (f32(2.0 ** -126), 1.0),        # M normal, M/2 subnormal: IEEE division path
    (f32(1.5e-40), 1.0),            # subnormal M: IEEE division path
    (f32(7.0e-45), 1.9),            # tiny subnormal
    (np.finfo(f32).max / f32(2.5), 1.9),
]


def _band(center, width=1 << 16):
    c = np.array([center], f32).view(np.int32)[0]
    bits = np.arange(max(c - width, 0), c + width, dtype=np.int64)
    bits = bits[(bits >= 0) & (bits < 0x7f800000)].astype(np.int32)
    return bits.view(f32)


def _check(T, t, s):
    import torch

    n = t.size
    td = torch.from_numpy(t).cuda()
    ed = torch.zeros(n, device="cuda")
    payload, hdr = T.tlc_compress(td, ed, s, use_zre=False)
    torch.cuda.synchronize()
    buf = np.zeros(n, f32)
    c = O.compress(t, buf, s, False)
    h = T.parse_header(hdr)
    assert h["status"] == c.status == 0
    assert np.float32(h["M"]).view(np.uint32) == c.M.view(np.uint32)
    np.testing.assert_array_equal(payload[: c.payload_len].cpu().numpy(), c.payload)
    assert np.array_equal(ed.cpu().numpy().view(np.uint32), buf.view(np.uint32))
    return c.M


@pytest.mark.parametrize("a,s", REGIMES)
def test_decision_bands(a, s):
    import paper_1802_07389_b200 as T

    M = f32(a) * f32(s)
    half = M / f32(2) if M / f32(2) > 0 else f32(0)
    parts = [_band(half), _band(M)]
    vals = np.concatenate(parts)
    vals = vals[np.abs(vals) <= a]
    g = synth.rng(123)
    rnd = (g.uniform(-1, 1, 200_000) * float(a)).astype(f32)
    t = np.concatenate([vals, -vals, rnd, np.array([a], f32)])
    g.shuffle(t)
    assert _check(T, t, s) == M


@pytest.mark.skipif(os.environ.get("TLC_EXHAUSTIVE") != "1", reason="set TLC_EXHAUSTIVE=1")
def test_exhaustive_unit_scale():
    import paper_1802_07389_b200 as T

    top = int(np.array([1.0], f32).view(np.int32)[0])
    chunk = 1 << 27
    for lo in range(0, top + 1, chunk):
        bits = np.arange(lo, min(lo + chunk, top + 1), dtype=np.int64).astype(np.int32)
        v = bits.view(f32)
        t = np.concatenate([v, -v, np.array([1.0], f32)])
        _check(T, t, 1.0)
