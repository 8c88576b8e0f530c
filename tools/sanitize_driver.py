"""Every kernel of libtlc once at small sizes, for compute-sanitizer (memcheck, racecheck,
synccheck): K1-K5 over single tensors and tables (ragged sizes, several K3/K4 chunks and
K5 tiles), the bulk-copy K2 paths, K6/K7 and the cooperative K6c, corrupt payloads
(FORMAT: nothing may be written outside out[0, n)), NaN input, Stoch 3-value + QE, 8-bit
int, the loopback exchange (K4 + K5m over several sources, the apply), tlc_aggregate,
and (MODE=full) a W=1 peer-memory exchange with its flag barrier.  Exits 0 when every
result is as expected; the sanitizer reports errors separately."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1802_07389_b200 as T  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda", 0)
full = os.environ.get("MODE", "full") == "full"


def codec(n, s, zre, family="gauss", off=0):
    t = torch.from_numpy(synth.family(family, n, s) if family != "gauss" else synth.gaussian(n, 5, n)).to(dev)
    base = torch.zeros(n + off, device=dev)
    err = base[off:]
    err.zero_()
    p, h = T.tlc_compress(t, err, s, zre)
    out = T.tlc_decompress(p, h, n)
    acc = torch.zeros(n, device=dev)
    T.tlc_decompress(p, h, n, acc, T.TLC_MODE_ACCUMULATE)
    torch.cuda.synchronize()
    hd = T.parse_header(h)
    assert hd["status"] == 0, hd
    return p, h, hd


for n in (1, 7, 1000, 4099, 65537, 300_001):
    for zre in (True, False):
        codec(n, 1.75, zre)
codec(300_000, 1.0, True, "dense")
codec(300_000, 1.75, True, "runs")
codec(300_000, 1.75, True, "zeros")
codec(300_000, 1.5, True, off=1)                              # misaligned err: scalar K2 path
# corrupt payloads: FORMAT, and no byte of `out` beyond n written (canary tail)
p, h, hd = codec(300_001, 1.75, True)
n = 300_001
for bad in ("truncate", "overrun", "literal"):
    q = p.clone()
    hh = h.clone()
    if bad == "truncate":
        hh[16:24] = torch.tensor(list(int(hd["payload_len"] - 3).to_bytes(8, "little")), dtype=torch.uint8)
    elif bad == "overrun":
        q[int((q[: hd["payload_len"]] < 243).nonzero()[0])] = 255     # a literal becomes a 14-run code
    else:
        hh[4] = 0                                               # claim no ZRE: bytes > 242 are invalid
        hh[16:24] = torch.tensor(list(int(-(-n // 5)).to_bytes(8, "little")), dtype=torch.uint8)
        q[: -(-n // 5)] = 250
    big = torch.full((n + 4096,), 7.0, device=dev)
    T.tlc_decompress(q, hh, n, big[:n])
    torch.cuda.synchronize()
    assert T.parse_header(hh)["status"] == T.TLC_ERR_FORMAT, bad
    assert bool((big[n:] == 7.0).all()), bad
# NaN input: NONFINITE, err untouched
t = torch.from_numpy(synth.gaussian(5000, 6)).to(dev)
t[100] = float("nan")
err = torch.full((5000,), 0.25, device=dev)
p, h = T.tlc_compress(t, err, 1.5, True)
torch.cuda.synchronize()
assert T.parse_header(h)["status"] == T.TLC_ERR_NONFINITE and bool((err == 0.25).all())
# tables: small (K6/K7, and K6c under TLC_COOP=1) and streaming
for sizes in (synth.RESNET110_SIZES[:40], [70_000, 3, 100_001, 40_960, 5]):
    ts = T.TensorSet(sizes, dev)
    xs = [torch.from_numpy(synth.gaussian(k, 8, i)).to(dev) for i, k in enumerate(sizes)]
    outs = [torch.empty(k, device=dev) for k in sizes]
    for _ in range(2):
        ts.compress(xs, 1.75, True)
        ts.decompress(outs)
        ts.decompress(outs, T.TLC_MODE_ACCUMULATE)
    torch.cuda.synchronize()
    assert all(hd["status"] == 0 for hd in ts.headers())
# compared designs
t = torch.from_numpy(synth.gaussian(200_003, 9)).to(dev)
p, h = T.tlc_stoch_compress(t, 1, 2, True)
T.tlc_decompress(p, h, t.numel())
c, h8 = T.tlc_int8_compress(t)
T.tlc_int8_decompress(c, h8, t.numel())
torch.cuda.synchronize()
# loopback exchange: K4 + K5m over 3 sources, pull compress, apply
sizes = [432, 9216, 36864, 200_003]
g = T.Loopback(3, sizes, dev)
grads = [[torch.from_numpy(synth.gaussian(k, 10, r, i)).to(dev) for i, k in enumerate(sizes)] for r in range(3)]
outs = [[torch.zeros(k, device=dev) for k in sizes] for _ in range(3)]
for _ in range(2):
    g.push(grads, 1.9)
    g.pull(outs, 1.9)
torch.cuda.synchronize()
assert all(x.status() == 0 for x in g.ranks)
g.close()
if full:
    comm = T.Comm(0, 1, dev)
    x = T.Exchange(comm, sizes, p2p=True)                     # flag barrier kernel (W = 1)
    o1 = [torch.zeros(k, device=dev) for k in sizes]
    for _ in range(2):
        x.push(grads[0], 1.75)
        x.pull(o1, 1.75)
    assert x.status() == 0
    x.close()
    comm.close()
torch.cuda.synchronize()
print("sanitize driver ok")
