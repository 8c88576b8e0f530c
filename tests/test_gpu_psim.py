"""The desk-scale training simulator (SPEC psim S:424-515) on a GPU.

* parity: every step's server means and the workers' replica after the shared pull are
  bitwise equal to the oracle (oracle.compress / decompress per worker and tensor, rank-order
  fold from +0, / W; one pull compression per tensor) run on the recorded gradients / deltas;
* S:609 acceptance: average bits per state change non-increasing in s; No-ZRE = 1.60 bits
  exactly (Table 2) when tensor sizes are multiples of 5;
* convergence sanity: 3LC s = 1 reaches the uncompressed run's test accuracy
  within a few points on the blob task.
"""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu
f32 = np.float32


@pytest.fixture(scope="module")
def psim():
    import torch

    assert torch.cuda.is_available()
    from paper_1802_07389_b200 import psim

    return psim


@pytest.mark.parametrize("W,s,zre", [(1, 1.0, True), (3, 1.5, True), (4, 1.9, False)])
def test_sim_parity_with_oracle(psim, W, s, zre):
    cfg = psim.SimConfig(workers=W, steps=4, s=s, use_zre=zre, input_dim=33, hidden=47, classes=7,
                         n_train=1024, n_test=128, eval_every=0)
    sim = psim.Sim(cfg)
    comp = sim.comp
    push_err = [[np.zeros(n, f32) for n in sim.sizes] for _ in range(W)]
    pull_err = [np.zeros(n, f32) for n in sim.sizes]
    rep = [sim.replica[i].cpu().numpy().reshape(-1).copy() for i in comp]
    for _ in range(cfg.steps):
        rec, grads, means, deltas = sim.step(record=True)
        bytes_push = 0
        for k, i in enumerate(comp):
            acc = np.zeros(sim.sizes[k], f32)
            for w in range(W):
                g = grads[w][i].cpu().numpy()
                c = O.compress(g, push_err[w][k], s, zre)
                assert c.status == O.OK
                bytes_push += c.payload_len
                st, acc = O.decompress(c.payload, zre, c.M, g.size, out=acc, accumulate=True)
                assert st == O.OK
            mean = (acc / f32(W)).astype(f32)
            assert np.array_equal(means[k].cpu().numpy().view(np.uint32), mean.view(np.uint32))
            d = deltas[i].cpu().numpy()
            c = O.compress(d, pull_err[k], s, zre)
            st, rep[k] = O.decompress(c.payload, zre, c.M, d.size, out=rep[k], accumulate=True)
            assert st == O.OK
            assert np.array_equal(sim.replica[i].cpu().numpy().reshape(-1).view(np.uint32), rep[k].view(np.uint32))
        assert rec["push_bytes_total"] == bytes_push


def test_bits_monotone_in_s_and_no_zre_density(psim):
    base = dict(workers=4, steps=80, input_dim=60, hidden=250, classes=10, n_train=4096, n_test=512, eval_every=0)
    bits = []
    for s in (1.0, 1.5, 1.75, 1.9):
        log = psim.Sim(psim.SimConfig(s=s, **base)).run()
        bits.append(psim.summarize(log, 1.0)["bits_per_value_push_all"])
    assert all(a >= b for a, b in zip(bits, bits[1:])), bits
    log = psim.Sim(psim.SimConfig(s=1.0, use_zre=False, **base)).run()
    assert all(r["bits_per_value_push"] == 1.6 and r["bits_per_value_pull"] == 1.6 for r in log)


def test_convergence_close_to_uncompressed(psim):
    base = dict(workers=4, steps=300, eval_every=100)
    ref = psim.summarize(psim.Sim(psim.SimConfig(codec="none", **base)).run())
    tlc = psim.summarize(psim.Sim(psim.SimConfig(codec="3lc", s=1.0, **base)).run())
    assert ref["final_test_acc"] > 0.8, ref
    assert tlc["final_test_acc"] >= ref["final_test_acc"] - 0.05, (tlc, ref)
    for codec in ("stoch", "int8"):
        r = psim.summarize(psim.Sim(psim.SimConfig(codec=codec, **base)).run())
        assert np.isfinite(r["final_loss"])
