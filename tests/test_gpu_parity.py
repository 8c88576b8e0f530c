"""GPU (sm_100a, through the C ABI) vs the CPU oracle, element by element.

Bar (north_star): bit-exact payload bytes (quartic + ZRE stream), header, and
bitwise-identical fp32 error buffer and decompressed tensor (0 ulp).
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


def _dev(x, offset=0):
    """Copy a numpy fp32 array to the GPU, optionally `offset` elements into a
    larger allocation so the kernels see a misaligned base pointer."""
    import torch

    buf = torch.empty(x.size + offset + 4, dtype=torch.float32, device="cuda")
    v = buf[offset:offset + x.size]
    v.copy_(torch.from_numpy(np.ascontiguousarray(x)))
    return v


def gpu_roundtrip(T, t, err0, s, use_zre, offset=0, acc_base=None):
    import torch

    n = t.size
    td, ed = _dev(t, offset), _dev(err0, offset)
    payload, hdr = T.tlc_compress(td, ed, s, use_zre)
    torch.cuda.synchronize()
    h = T.parse_header(hdr)
    res = {"hdr": h, "err": ed.cpu().numpy(), "payload": payload[: h["payload_len"]].cpu().numpy()}
    if h["status"] == 0:
        out = _dev(np.zeros(n, f32), offset)
        T.tlc_decompress(payload, hdr, n, out)
        torch.cuda.synchronize()
        res["out"] = out.cpu().numpy()
        res["dstatus"] = T.parse_header(hdr)["status"]
        if acc_base is not None:
            acc = _dev(acc_base, offset)
            T.tlc_decompress(payload, hdr, n, acc, mode=T.TLC_MODE_ACCUMULATE)
            torch.cuda.synchronize()
            res["acc"] = acc.cpu().numpy()
    return res


def check_case(T, t, err0, s, use_zre, offset=0):
    n = t.size
    g = synth.rng(99, n)
    acc_base = g.standard_normal(n).astype(f32)
    acc_base[::7] = f32(-0.0)
    r = gpu_roundtrip(T, t, err0, s, use_zre, offset, acc_base)
    buf = err0.copy()
    c = O.compress(t, buf, s, use_zre)
    h = r["hdr"]
    assert h["status"] == c.status
    assert h["n"] == n
    if c.status != O.OK:
        assert np.array_equal(r["err"].view(np.uint32), err0.view(np.uint32))
        return r
    assert np.float32(h["M"]).view(np.uint32) == c.M.view(np.uint32)
    assert h["flags"] == (1 if use_zre else 0)
    assert h["payload_len"] == c.payload_len, (n, s, use_zre)
    np.testing.assert_array_equal(r["payload"], c.payload)
    assert np.array_equal(r["err"].view(np.uint32), buf.view(np.uint32)), "err buffer not bitwise equal"
    st, out = O.decompress(c.payload, use_zre, c.M, n)
    assert st == O.OK and r["dstatus"] == 0
    assert np.array_equal(r["out"].view(np.uint32), out.view(np.uint32)), "decompressed not bitwise equal"
    st, acc = O.decompress(c.payload, use_zre, c.M, n, out=acc_base.copy(), accumulate=True)
    assert np.array_equal(r["acc"].view(np.uint32), acc.view(np.uint32)), "accumulate not bitwise equal"
    return r


SIZES_SMALL = list(range(1, 51)) + [
    # n = 5P - k, k = 0..4, P = 0..7 mod 8 around one and two K2 tiles (2048 bytes)
    *[5 * P - k for P in (2040, 2043, 2047, 2048, 2049, 2050, 4095, 4096, 4097) for k in (0, 3, 4)],
    70, 71, 1000, 70_000, 123_457, 1 << 20, (1 << 20) + 3,
]


@pytest.mark.parametrize("family", ["gauss", "zeros", "dense", "runs"])
@pytest.mark.parametrize("use_zre", [True, False])
def test_parity_sizes(tlc, family, use_zre):
    for n in SIZES_SMALL:
        for s in (1.0, 1.75):
            t = synth.family(family, n, s, seed=3 + n)
            err0 = np.zeros(n, f32) if family != "gauss" else (0.3 * synth.gaussian(n, 4, n)).astype(f32)
            check_case(tlc, t, err0, s, use_zre)


@pytest.mark.parametrize("offset", [1, 2, 3])
def test_parity_misaligned(tlc, offset):
    """Base pointers not 16-byte aligned -> the scalar load/store paths."""
    for n in (1, 7, 4099, 10_241, 100_003, 1 << 18):
        t = synth.gaussian(n, 5, n)
        err0 = (0.5 * synth.gaussian(n, 6, n)).astype(f32)
        check_case(tlc, t, err0, 1.9, True, offset=offset)
        check_case(tlc, t, err0, 1.0, False, offset=offset)


@pytest.mark.parametrize("pmod", [0, 1, 2, 3])
def test_parity_bulk_partition_alignment(tlc, pmod):
    """Single tensors large enough for the bulk-copy (TMA) K2 path, with P = ceil(n/5) in every
    residue mod 4: P % 4 != 0 makes every partition after the first start off a 16-byte
    boundary (aligned-superset copies shifted by (i P) mod 4)."""
    for base in (5 * 4096 * 4, 5 * 4096 * 37, 1 << 22):
        P = -(-base // 5)
        P += (pmod - P) % 4
        for k in (0, 3):
            n = 5 * P - k
            t = synth.gaussian(n, 8, n)
            err0 = (0.4 * synth.gaussian(n, 9, n)).astype(f32)
            check_case(tlc, t, err0, 1.75, True)
            check_case(tlc, t, err0, 1.0, False)


def test_parity_runs_many_tiles(tlc):
    """Runs of 121 bytes (lengths 1..100, 14k+-1) crossing many tile edges."""
    for n in (5 * 2048 * 7 + 3, 5 * 2048 * 64, 999_999, 3_000_001):
        for s in (1.0, 1.5, 1.9):
            t = synth.runs_adversarial(n, 1.0, 21, n)
            check_case(tlc, t, np.zeros(n, f32), s, True)


def test_parity_error_feedback_steps(tlc):
    """K error-feedback steps on both sides, err compared bitwise every step."""
    import torch

    T = tlc
    n = 300_007
    ed = _dev(np.zeros(n, f32))
    buf = np.zeros(n, f32)
    for step in range(6):
        t = synth.gaussian(n, 31, step)
        td = _dev(t)
        payload, hdr = T.tlc_compress(td, ed, 1.75, True)
        torch.cuda.synchronize()
        h = T.parse_header(hdr)
        c = O.compress(t, buf, 1.75, True)
        assert h["payload_len"] == c.payload_len
        np.testing.assert_array_equal(payload[: h["payload_len"]].cpu().numpy(), c.payload)
        assert np.array_equal(ed.cpu().numpy().view(np.uint32), buf.view(np.uint32))


def test_special_values(tlc):
    """-0 inputs, subnormal M (division path), tiny and huge magnitudes."""
    n = 5000
    g = synth.rng(41)
    cases = []
    t = np.zeros(n, f32)
    t[::3] = f32(-0.0)
    t[17] = f32(1e-3)
    cases.append(t)
    # subnormal max -> M < 2^-125 uses IEEE division
    t = (g.standard_normal(n) * 1e-40).astype(f32)
    cases.append(t)
    t = (g.standard_normal(n) * 1e-39).astype(f32)
    cases.append(t)
    t = (g.standard_normal(n) * 1e30).astype(f32)
    cases.append(t)
    # exact ties at M/2: u = +-M/2 and neighbours
    t = np.zeros(n, f32)
    t[0] = f32(3.0)
    t[1:10] = [1.5, -1.5, np.nextafter(f32(1.5), f32(0)), -np.nextafter(f32(1.5), f32(0)), 1.5, 0, -0.0, 3.0, -3.0]
    cases.append(t)
    for t in cases:
        for s in (1.0, 1.5, 1.9):
            err0 = np.zeros(n, f32)
            err0[::5] = f32(-0.0)
            check_case(tlc, t, err0, s, True)
            check_case(tlc, t, err0, s, False)


def test_nonfinite_and_range(tlc):
    n = 10_000
    for bad, code, s in ((np.nan, 2, 1.0), (np.inf, 2, 1.0), (-np.inf, 2, 1.5), (np.finfo(f32).max, 3, 1.5)):
        for pos in (0, n // 2, n - 1):
            t = synth.gaussian(n, 51, pos)
            t[pos] = bad
            err0 = (0.1 * synth.gaussian(n, 52, pos)).astype(f32)
            r = check_case(tlc, t, err0, s, True)
            assert r["hdr"]["status"] == code


def test_argument_errors(tlc):
    import torch

    T = tlc
    t = torch.zeros(10, device="cuda")
    e = torch.zeros(10, device="cuda")
    for s in (0.5, 2.0, float("nan")):
        with pytest.raises(T.TlcError) as ei:
            T.tlc_compress(t, e, s)
        assert ei.value.code == T.TLC_ERR_ARG
    small = torch.empty(1, dtype=torch.uint8, device="cuda")
    with pytest.raises(T.TlcError) as ei:
        T.tlc_compress(t, e, 1.0, payload=small)
    assert ei.value.code == T.TLC_ERR_CAPACITY


def test_corrupt_payloads_raise_format(tlc):
    import torch

    T = tlc
    n = 70 * 50
    t = np.zeros(n, f32)
    td, ed = _dev(t), _dev(np.zeros(n, f32))
    payload, hdr = T.tlc_compress(td, ed, 1.0, True)
    torch.cuda.synchronize()
    good = T.parse_header(hdr)
    assert good["payload_len"] == 50

    def run(mutate_payload=None, mutate_hdr=None, n_arg=n):
        p = payload.clone()
        h = hdr.clone()
        if mutate_payload:
            mutate_payload(p)
        if mutate_hdr:
            mutate_hdr(h)
        out = torch.zeros(n + 64, device="cuda")
        T.tlc_decompress(p, h, n_arg, out[:n_arg])
        torch.cuda.synchronize()
        assert torch.all(out[n_arg:] == 0), "wrote past the end of out"
        return T.parse_header(h)["status"]

    import struct

    def set_len(v):
        def f(h):
            h[16:24] = torch.tensor(list(struct.pack("<Q", v)), dtype=torch.uint8)
        return f

    assert run() == 0
    assert run(mutate_hdr=set_len(49)) == T.TLC_ERR_FORMAT          # truncated
    assert run(mutate_payload=lambda p: p.__setitem__(0, 121)) == T.TLC_ERR_FORMAT  # short by 13
    big = payload.clone()
    assert run(mutate_payload=lambda p: p.__setitem__(slice(0, 50), 255), mutate_hdr=set_len(51)) == T.TLC_ERR_FORMAT
    assert run(n_arg=n - 5) == T.TLC_ERR_FORMAT                      # hdr.n mismatch

    def set_M(v):
        def f(h):
            h[0:4] = torch.tensor(list(struct.pack("<f", v)), dtype=torch.uint8)
        return f

    for bad_M in (-1.0, -0.0, float("nan"), float("inf")):                # R21
        assert run(mutate_hdr=set_M(bad_M)) == T.TLC_ERR_FORMAT

    # no-ZRE stream with a literal > 242
    td2, ed2 = _dev(synth.gaussian(1000, 61)), _dev(np.zeros(1000, f32))
    p2, h2 = T.tlc_compress(td2, ed2, 1.0, False)
    p2[5] = 250
    out = torch.zeros(1000, device="cuda")
    T.tlc_decompress(p2, h2, 1000, out)
    torch.cuda.synchronize()
    assert T.parse_header(h2)["status"] == T.TLC_ERR_FORMAT


def test_full_size_headline_config(tlc):
    """BASELINE config C3: n = 2^28, s = 1.75, gauss-steady (error feedback),
    launched exactly as bench.py launches it; full element-wise comparison."""
    import torch

    T = tlc
    n = 1 << 28
    t = synth.gaussian(n, 3, 0)
    td = _dev(t)
    ed = _dev(np.zeros(n, f32))
    buf = np.zeros(n, f32)
    for step in range(2):
        payload, hdr = T.tlc_compress(td, ed, 1.75, True)
        c = O.compress(t, buf, 1.75, True)
        torch.cuda.synchronize()
        h = T.parse_header(hdr)
        assert h["status"] == 0 and h["payload_len"] == c.payload_len
        np.testing.assert_array_equal(payload[: h["payload_len"]].cpu().numpy(), c.payload)
        assert torch.equal(ed.view(torch.int32).cpu(), torch.from_numpy(buf.view(np.int32)))
    out = torch.empty(n, device="cuda")
    T.tlc_decompress(payload, hdr, n, out)
    st, ref = O.decompress(c.payload, True, c.M, n)
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int32).cpu(), torch.from_numpy(ref.view(np.int32)))
