"""tlc_aggregate (the server's fused "average the gradients") on its own: W
payload sets made by the CPU oracle are aggregated on the GPU and compared bit for bit with
the oracle's X3 (rank-ordered fold from +0 of the nonzero dequantized trits, IEEE / W,
R15); a source whose header carries a failure makes its tensor's mean NaN (R24)."""
import numpy as np
import pytest

import oracle as O
import synth

pytestmark = pytest.mark.gpu
f32 = np.float32


@pytest.mark.parametrize("W", [1, 2, 3, 5, 8])
@pytest.mark.parametrize("s,zre", [(1.0, True), (1.9, True), (1.5, False)])
def test_aggregate_matches_oracle_fold(W, s, zre):
    import torch

    import paper_1802_07389_b200 as T

    dev = torch.device("cuda", 0)
    sizes = [5, 1000, 36864, 20003, 70]
    srcs, ref = [], []
    sent = []
    for w in range(W):
        pays, hdrs, row = [], [], []
        for i, n in enumerate(sizes):
            t = (synth.gaussian(n, 41, w, i) * f32(1.7 ** w)).astype(f32)
            if i == 4:
                t[:] = 0.0                                          # an all-zero tensor (M = 0)
            c = O.compress(t, np.zeros(n, f32), s, zre)
            row.append(c)
            p = torch.zeros(max(1, T.tlc_max_payload_bytes(n)), dtype=torch.uint8, device=dev)
            p[: c.payload_len] = torch.from_numpy(c.payload).to(dev)
            h = T.Header(float(c.M), 1 if zre else 0, n, c.payload_len, 0, 0)
            hb = torch.frombuffer(bytearray(bytes(h)), dtype=torch.uint8).to(dev)
            pays.append(p)
            hdrs.append(hb)
        srcs.append((pays, hdrs))
        sent.append(row)
    outs = [torch.full((n,), float("nan"), device=dev) for n in sizes]
    agg = T.Aggregate(outs, srcs)
    agg.run()
    torch.cuda.synchronize()
    for i, n in enumerate(sizes):
        acc = np.zeros(n, f32)
        for w in range(W):
            st, acc = O.decompress(sent[w][i].payload, zre, sent[w][i].M, n, out=acc, accumulate=True)
            assert st == 0
        mean = (acc / f32(W)).astype(f32)
        assert np.array_equal(outs[i].cpu().numpy().view(np.uint32), mean.view(np.uint32)), (W, i)
    # R24: mark one source of tensor 1 as failed -> NaN mean for tensor 1 only
    bad = srcs[W - 1][1][1]
    bad[24:28] = torch.tensor([2, 0, 0, 0], dtype=torch.uint8, device=dev)      # status = NONFINITE
    agg.run()
    torch.cuda.synchronize()
    assert torch.isnan(outs[1]).all()
    assert not torch.isnan(outs[0]).any() and not torch.isnan(outs[2]).any()
    agg.close()
