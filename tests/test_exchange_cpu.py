"""CPU checks of the exchange (row e): the library's plan against the oracle's
independent plan (R17), plan invariants, and the W-virtual-rank oracle's
properties (W=1 reduces to compress/decompress, replicas stay identical)."""
import numpy as np
import pytest

import oracle as O
import synth
from oracle import exchange as X

f32 = np.float32

SIZE_LISTS = [
    synth.RESNET110_SIZES, synth.RESNET50_SIZES, synth.BERT_LARGE_SIZES,
    [100, 3, 3], [7], [1, 1, 1, 1, 1], [10 ** 6, 5, 10 ** 6 + 1, 2], [0, 5, 0, 9],
]


@pytest.fixture(scope="module")
def T():
    import __graft_entry__

    __graft_entry__.build()        # builds libtlc.so on a fresh checkout (no package import first)
    import paper_1802_07389_b200 as T

    return T


@pytest.mark.parametrize("W", [1, 2, 3, 4, 5, 8])
def test_plan_matches_oracle(T, W):
    for sizes in SIZE_LISTS:
        assert T.tlc_plan(sizes, W) == X.plan(sizes, W)


@pytest.mark.parametrize("W", [1, 2, 4, 8])
def test_plan_invariants(W):
    for sizes in SIZE_LISTS:
        ctx = X.plan(sizes, W)
        N = sum(sizes)
        cap = max(1, -(-N // W))
        for t, n in enumerate(sizes):
            parts = sorted((lo, hi) for (tt, lo, hi, _) in ctx if tt == t)
            if n == 0:
                assert parts == []
                continue
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))          # contiguous cover
            lens = [hi - lo for lo, hi in parts]
            assert max(lens) - min(lens) <= 1 and max(lens) <= max(cap, 1)   # equal shards <= cap
        assert all(0 <= o < W for (_, _, _, o) in ctx)


def test_virtual_ps_w1_is_compress_decompress():
    """X1-X6 with W = 1: the mean is the dequantized push, the pull adds the
    dequantized compression of that mean."""
    sizes = [1000, 4099, 70]
    ps = X.VirtualPS(sizes, 1)
    grads = [[synth.gaussian(n, 81, t) for t, n in enumerate(sizes)]]
    outs = [[np.zeros(n, f32) for n in sizes]]
    means, sent, shared = ps.step(grads, outs, 1.75)
    for c, (t, lo, hi, _) in enumerate(ps.ctx):
        buf = np.zeros(hi - lo, f32)
        cp = O.compress(grads[0][t][lo:hi], buf, 1.75)
        st, dq = O.decompress(cp.payload, True, cp.M, hi - lo)
        assert np.array_equal(means[c], dq)
        buf2 = np.zeros(hi - lo, f32)
        cp2 = O.compress(dq, buf2, 1.75)
        st, dq2 = O.decompress(cp2.payload, True, cp2.M, hi - lo)
        assert np.array_equal(outs[0][t][lo:hi], dq2)


def test_virtual_ps_replicas_identical_and_conservation():
    sizes = synth.RESNET110_SIZES[:12]
    W = 4
    ps = X.VirtualPS(sizes, W)
    outs = [[np.zeros(n, f32) for n in sizes] for _ in range(W)]
    total_mean = [np.zeros(n, np.float64) for n in sizes]
    for step in range(3):
        grads = [[synth.gaussian(n, 82, r, t, step) for t, n in enumerate(sizes)] for r in range(W)]
        means, _, _ = ps.step(grads, outs, 1.5)
        for c, (t, lo, hi, _) in enumerate(ps.ctx):
            total_mean[t][lo:hi] += means[c]
    for r in range(1, W):
        for t in range(len(sizes)):
            assert np.array_equal(outs[r][t].view(np.uint32), outs[0][t].view(np.uint32))
    # pull telescoping: applied deltas + pull error buffers == sum of the means (fp32 rounding)
    for c, (t, lo, hi, _) in enumerate(ps.ctx):
        lhs = outs[0][t][lo:hi].astype(np.float64) + ps.pull_err[c]
        assert np.allclose(lhs, total_mean[t][lo:hi], atol=1e-4)
