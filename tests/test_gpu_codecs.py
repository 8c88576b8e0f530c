"""GPU vs oracle for the compared designs of Sec. 5.1, through the C ABI:
"Stoch 3-value + QE" (tlc_stoch_compress, reading R22) and "8-bit int"
(tlc_int8_compress / tlc_int8_decompress, reading R23).

Bar: header, payload / code bytes bit-exact; decompressed fp32 bitwise equal (0 ulp).
"""
import numpy as np
import pytest

import oracle as O
import synth

pytestmark = pytest.mark.gpu

f32 = np.float32


@pytest.fixture(scope="module")
def tlc():
    import torch

    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    import paper_1802_07389_b200 as T

    return T


def _dev(x, offset=0, dtype=None):
    import torch

    x = np.ascontiguousarray(x)
    tdt = {np.float32: torch.float32, np.int8: torch.int8}[x.dtype.type]
    buf = torch.empty(x.size + offset + 16, dtype=tdt, device="cuda")
    v = buf[offset:offset + x.size]
    v.copy_(torch.from_numpy(x))
    return v


# --------------------------------------------------------------------------- stochastic 3-value + QE
def stoch_case(T, t, seed, step, use_zre, offset=0):
    import torch

    n = t.size
    td = _dev(t, offset)
    payload, hdr = T.tlc_stoch_compress(td, seed, step, use_zre)
    torch.cuda.synchronize()
    h = T.parse_header(hdr)
    c = O.stoch_compress(t, seed, step, use_zre)
    assert h["status"] == c.status, (n, h)
    assert h["n"] == n
    if c.status != O.OK:
        return
    assert f32(h["M"]).view(np.uint32) == c.M.view(np.uint32)
    assert h["flags"] == (1 if use_zre else 0)
    assert h["payload_len"] == c.payload_len, (n, seed, step, use_zre)
    np.testing.assert_array_equal(payload[: h["payload_len"]].cpu().numpy(), c.payload)
    out = T.tlc_decompress(payload, hdr, n)
    torch.cuda.synchronize()
    st, ref = O.decompress(c.payload, use_zre, c.M, n)
    assert st == O.OK and T.parse_header(hdr)["status"] == 0
    assert np.array_equal(out.cpu().numpy().view(np.uint32), ref.view(np.uint32))


@pytest.mark.parametrize("use_zre", [False, True])
def test_stoch_sizes(tlc, use_zre):
    for n in list(range(1, 51)) + [1023, 1024, 1025, 5 * 1024 * 4 - 1, 5 * 4096 + 3, 100_003, (1 << 20) + 7]:
        t = synth.gaussian(n, 71, n)
        stoch_case(tlc, t, seed=1000 + n, step=n % 7, use_zre=use_zre)


def test_stoch_tile_edges_and_big_counters(tlc):
    """P around the 1K / 4K tile sizes with every n mod 5, and 64-bit seeds / steps (both
    halves of the Philox counter and key in use)."""
    for P in [1023, 1024, 1025, 2047, 4095, 4096, 4097, 8191, 12289]:
        for k in range(5):
            n = 5 * P - k
            t = synth.gaussian(n, 72, n)
            stoch_case(tlc, t, seed=0xFEDCBA9876543210 + k, step=(3 << 32) + P, use_zre=(k % 2 == 0))


@pytest.mark.parametrize("offset", [1, 2, 3])
def test_stoch_misaligned(tlc, offset):
    for n in [7, 333, 4096 * 5 + 1, 65537]:
        stoch_case(tlc, synth.gaussian(n, 73, n), seed=5, step=2, use_zre=True, offset=offset)


def test_stoch_special_values(tlc):
    n = 20_011
    g = synth.rng(74)
    t = g.standard_normal(n).astype(f32)
    t[::13] = f32(0.0)
    t[1::17] = f32(-0.0)
    t[5] = f32(-7.5)                        # the max: always -1
    t[6::31] = f32(3.75)                    # |x|/m = 1/2 exactly
    t[7::37] = np.float32(1e-40)            # subnormal: p = fl(1e-40/7.5) (tiny)
    stoch_case(tlc, t, 9, 4, True)
    stoch_case(tlc, np.zeros(n, f32), 9, 4, True)           # m = 0: all digits 1
    for bad in (np.nan, np.inf, -np.inf):
        tb = t.copy()
        tb[n // 2] = bad
        stoch_case(tlc, tb, 9, 4, False)                    # NONFINITE


def test_stoch_full_size(tlc):
    """The bench configuration (n = 2^28, QE only as the paper's design): every payload byte."""
    import torch

    n = 1 << 28
    t = synth.gaussian(n, 3, 0)
    td = torch.from_numpy(t).cuda()
    payload, hdr = tlc.tlc_stoch_compress(td, 12345, 1, False)
    torch.cuda.synchronize()
    h = tlc.parse_header(hdr)
    del td
    c = O.stoch_compress(t, 12345, 1, False)
    assert h["status"] == 0 and h["payload_len"] == c.payload_len
    assert f32(h["M"]) == c.M
    assert np.array_equal(payload[: c.payload_len].cpu().numpy(), c.payload)


# --------------------------------------------------------------------------- 8-bit int
def int8_case(T, t, offset=0, acc_base=None):
    import torch

    n = t.size
    td = _dev(t, offset)
    codes = _dev(np.zeros(n, np.int8), offset)
    codes, hdr = T.tlc_int8_compress(td, codes)
    torch.cuda.synchronize()
    h = T.parse_header(hdr)
    st, sc, ref_codes = O.int8_compress(t)
    assert h["status"] == st
    if st != O.OK:
        return
    assert h["flags"] == T.TLC_FLAG_INT8 and h["n"] == n and h["payload_len"] == n
    assert f32(h["M"]).view(np.uint32) == sc.view(np.uint32)
    np.testing.assert_array_equal(codes.cpu().numpy(), ref_codes)
    out = _dev(np.zeros(n, f32), offset)
    T.tlc_int8_decompress(codes, hdr, n, out)
    torch.cuda.synchronize()
    ref = O.int8_decompress(ref_codes, sc)
    assert np.array_equal(out.cpu().numpy().view(np.uint32), ref.view(np.uint32))
    if acc_base is not None:
        acc = _dev(acc_base, offset)
        T.tlc_int8_decompress(codes, hdr, n, acc, mode=T.TLC_MODE_ACCUMULATE)
        torch.cuda.synchronize()
        ref_acc = O.int8_decompress(ref_codes, sc, acc_base.copy(), accumulate=True)
        assert np.array_equal(acc.cpu().numpy().view(np.uint32), ref_acc.view(np.uint32))


def test_int8_sizes_and_offsets(tlc):
    for n in list(range(1, 40)) + [255, 256, 4097, 100_003, (1 << 20) + 5]:
        t = synth.gaussian(n, 81, n)
        base = synth.gaussian(n, 82, n)
        base[::5] = f32(-0.0)
        int8_case(tlc, t, 0, base)
    for off in (1, 2, 3, 5):
        n = 70_001
        int8_case(tlc, synth.gaussian(n, 83, off), off, synth.gaussian(n, 84, off))


def test_int8_ties_and_specials(tlc):
    t = np.array([127.0, 2.5, -2.5, 0.5, -0.5, 1.5, 126.5, -0.49999997, 0.0, -0.0] * 1000, dtype=f32)
    int8_case(tlc, t)                                    # scale 1: half away from zero
    int8_case(tlc, np.zeros(1000, f32))
    int8_case(tlc, np.array([1e-45, -1e-45, 0.0] * 33, dtype=f32))   # scale underflows (R23)
    g = synth.rng(85)
    t = (g.standard_normal(50_000) * 1e-38).astype(f32)               # subnormal quotients
    int8_case(tlc, t)
    for bad in (np.nan, np.inf):
        tb = synth.gaussian(1000, 86)
        tb[999] = bad
        int8_case(tlc, tb)


def test_int8_bad_header_is_format(tlc):
    import torch

    n = 1000
    td = _dev(synth.gaussian(n, 87))
    codes, hdr = tlc.tlc_int8_compress(td)
    out = torch.zeros(n + 16, dtype=torch.float32, device="cuda")
    tlc.tlc_int8_decompress(codes, hdr, n - 1, out[: n - 1])      # n mismatch
    torch.cuda.synchronize()
    assert tlc.parse_header(hdr)["status"] == tlc.TLC_ERR_FORMAT
    assert not out.any()
    payload, hdr2 = tlc.tlc_compress(td, torch.zeros(n, device="cuda"), 1.0, False)
    tlc.tlc_int8_decompress(codes, hdr2, n, out[:n])               # not an int8 header
    torch.cuda.synchronize()
    assert tlc.parse_header(hdr2)["status"] == tlc.TLC_ERR_FORMAT


def test_int8_full_size(tlc):
    import torch

    n = 1 << 28
    t = synth.gaussian(n, 3, 0)
    td = torch.from_numpy(t).cuda()
    codes, hdr = tlc.tlc_int8_compress(td)
    out = tlc.tlc_int8_decompress(codes, hdr, n)
    torch.cuda.synchronize()
    st, sc, ref_codes = O.int8_compress(t)
    assert np.array_equal(codes.cpu().numpy(), ref_codes)
    ref = O.int8_decompress(ref_codes, sc)
    assert np.array_equal(out.cpu().numpy().view(np.uint32), ref.view(np.uint32))
