"""Out-of-bounds write checks without compute-sanitizer (closed on this GPU pool): every
buffer the library writes -- err, payload, header, decompressed output, exchange outputs,
aggregate outputs, int8 codes -- lives between 4 KiB guard bands filled with a byte pattern,
and after each call the bands must be intact.  Covers K1-K5 on single tensors (ragged sizes,
misaligned views, several K3/K4 chunks and K5 tiles), corrupt payloads (FORMAT), the batched
small-table kernels (K6/K7, and K6c under TLC_COOP=1), the loopback exchange (K4 + K5m,
apply), tlc_aggregate and the compared designs."""
import os
import subprocess
import sys

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu
GUARD = 4096
PAT = 0xA5


class Guarded:
    """A device tensor of `n` elements of `dtype` at byte offset `off` (for misalignment)
    inside an allocation with GUARD pattern bytes on both sides."""

    def __init__(self, n, dtype, dev, off=0, fill=0):
        import torch

        es = torch.empty(0, dtype=dtype).element_size()
        self.raw = torch.full((2 * GUARD + n * es + off,), PAT, dtype=torch.uint8, device=dev)
        self.lo, self.hi = GUARD + off, GUARD + off + n * es
        self.t = self.raw[self.lo: self.hi].view(dtype)
        self.t.fill_(fill)

    def intact(self):
        r = self.raw.cpu().numpy()
        return bool((r[: self.lo] == PAT).all() and (r[self.hi:] == PAT).all())


def _dev():
    import torch

    return torch.device("cuda", 0)


@pytest.mark.parametrize("n,off", [(1, 0), (7, 4), (1000, 0), (4099, 8), (65537, 0), (300_001, 4), (1 << 20, 0)])
@pytest.mark.parametrize("zre", [True, False])
def test_codec_writes_stay_in_bounds(n, off, zre):
    import torch

    import paper_1802_07389_b200 as T

    dev = _dev()
    t = Guarded(n, torch.float32, dev, off)
    t.t.copy_(torch.from_numpy(synth.gaussian(n, 21, n)))
    err = Guarded(n, torch.float32, dev, off)
    pay = Guarded(T.tlc_max_payload_bytes(n), torch.uint8, dev, 1)
    hdr = Guarded(32, torch.uint8, dev)
    out = Guarded(n, torch.float32, dev, off)
    for s in (1.0, 1.75):
        T.tlc_compress(t.t, err.t, s, zre, pay.t, hdr.t)
        T.tlc_decompress(pay.t, hdr.t, n, out.t)
        T.tlc_decompress(pay.t, hdr.t, n, out.t, T.TLC_MODE_ACCUMULATE)
    torch.cuda.synchronize()
    assert T.parse_header(hdr.t)["status"] == 0
    assert all(g.intact() for g in (t, err, pay, hdr, out))


@pytest.mark.parametrize("bad", ["truncate", "overrun", "literal", "header_n"])
def test_corrupt_payloads_write_nothing_outside(bad):
    import torch

    import paper_1802_07389_b200 as T

    dev = _dev()
    n = 300_001
    t = torch.from_numpy(synth.gaussian(n, 22)).to(dev)
    pay, hdr = T.tlc_compress(t, torch.zeros(n, device=dev), 1.75, True)
    torch.cuda.synchronize()
    h = T.parse_header(hdr)
    P = -(-n // 5)
    if bad == "truncate":
        hdr[16:24] = torch.tensor(list(int(h["payload_len"] - 3).to_bytes(8, "little")), dtype=torch.uint8)
    elif bad == "overrun":
        k = int((pay[: h["payload_len"]] < 243).nonzero()[0])    # a literal becomes a 14-run code
        pay[k] = 255
    elif bad == "literal":
        hdr[4] = 0
        hdr[16:24] = torch.tensor(list(P.to_bytes(8, "little")), dtype=torch.uint8)
        pay[:P] = 250
    else:
        hdr[8:16] = torch.tensor(list((n + 5).to_bytes(8, "little")), dtype=torch.uint8)
    out = Guarded(n, torch.float32, dev)
    T.tlc_decompress(pay, hdr, n, out.t)
    torch.cuda.synchronize()
    assert T.parse_header(hdr)["status"] == T.TLC_ERR_FORMAT
    assert out.intact()


@pytest.mark.parametrize("coop", ["0", "1"])
def test_small_and_streaming_tables_in_bounds(coop):
    """Run in a subprocess so that TLC_COOP selects K6 or K6c for the small table."""
    code = f"""
import sys; sys.path[:0] = [{os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r}, {os.path.dirname(os.path.abspath(__file__))!r}]
import torch, synth
import paper_1802_07389_b200 as T
from test_gpu_guards import Guarded
dev = torch.device('cuda', 0)
for sizes in (synth.RESNET110_SIZES, [70_000, 3, 100_001, 40_960, 5, 36_864]):
    ts = [Guarded(k, torch.float32, dev, 4 * (i % 2)) for i, k in enumerate(sizes)]
    for i, g in enumerate(ts):
        g.t.copy_(torch.from_numpy(synth.gaussian(g.t.numel(), 23, i)))
    errs = [Guarded(k, torch.float32, dev) for k in sizes]
    pays = [Guarded(T.tlc_max_payload_bytes(k), torch.uint8, dev, 1) for k in sizes]
    hdrs = [Guarded(32, torch.uint8, dev) for k in sizes]
    outs = [Guarded(k, torch.float32, dev, 4) for k in sizes]
    b = T.Batch([(ts[i].t, errs[i].t, outs[i].t, pays[i].t, hdrs[i].t, k) for i, k in enumerate(sizes)])
    for s in (1.0, 1.9):
        b.compress(s, True)
        b.decompress(T.TLC_MODE_OVERWRITE)
        b.decompress(T.TLC_MODE_ACCUMULATE)
    torch.cuda.synchronize()
    for g in ts + errs + pays + hdrs + outs:
        assert g.intact()
print('ok')
"""
    env = dict(os.environ, TLC_COOP=coop)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]


@pytest.mark.parametrize("W", [2, 5])
def test_exchange_and_aggregate_in_bounds(W):
    import torch

    import paper_1802_07389_b200 as T

    dev = _dev()
    sizes = [432, 9216, 36864, 200_003]
    g = T.Loopback(W, sizes, dev)
    grads = [[Guarded(k, torch.float32, dev, 4 * (r % 2)) for k in sizes] for r in range(W)]
    for r in range(W):
        for i, x in enumerate(grads[r]):
            x.t.copy_(torch.from_numpy(synth.gaussian(x.t.numel(), 24, r, i)))
    outs = [[Guarded(k, torch.float32, dev, 4) for k in sizes] for _ in range(W)]
    for _ in range(2):
        g.push([[x.t for x in gr] for gr in grads], 1.5)
        g.pull([[o.t for o in orow] for orow in outs], 1.5)
    torch.cuda.synchronize()
    assert all(x.status() == 0 for x in g.ranks)
    assert all(o.intact() for orow in outs for o in orow) and all(x.intact() for gr in grads for x in gr)
    g.close()
    # the standalone aggregation into guarded outputs
    srcs = []
    for r in range(W):
        ts = T.TensorSet(sizes, dev)
        ts.compress([x.t for x in grads[r]], 1.5, True)
        srcs.append((ts.payloads, ts.hdrs))
    aouts = [Guarded(k, torch.float32, dev, 4) for k in sizes]
    agg = T.Aggregate([o.t for o in aouts], srcs)
    agg.run()
    torch.cuda.synchronize()
    assert all(o.intact() for o in aouts)


def test_compared_designs_in_bounds():
    import torch

    import paper_1802_07389_b200 as T

    dev = _dev()
    for n in (5, 4097, 200_003):
        t = torch.from_numpy(synth.gaussian(n, 25)).to(dev)
        pay = Guarded(T.tlc_max_payload_bytes(n), torch.uint8, dev, 1)
        hdr = Guarded(32, torch.uint8, dev)
        out = Guarded(n, torch.float32, dev, 4)
        T.tlc_stoch_compress(t, 3, 4, True, pay.t, hdr.t)
        T.tlc_decompress(pay.t, hdr.t, n, out.t)
        codes = Guarded(n, torch.int8, dev, 1)
        h8 = Guarded(32, torch.uint8, dev)
        T.tlc_int8_compress(t, codes.t, h8.t)
        T.tlc_int8_decompress(codes.t, h8.t, n, out.t)
        torch.cuda.synchronize()
        assert all(g.intact() for g in (pay, hdr, out, codes, h8))
