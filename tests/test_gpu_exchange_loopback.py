"""The multi-source exchange on ONE GPU: a loopback group (tlc_loopback_*) of W virtual
ranks runs the real push -> K5m -> pull -> apply kernels (K4 only under TLC_NO_PRODSEEK=1:
the consumers read the seek entries the producers' K3 wrote) -- every owner's fused
aggregation reading all W ranks' payloads, every rank's apply reading all owners'
payloads -- and is compared bit for bit with the W-virtual-rank oracle
(oracle/exchange.py, X1-X6): every owner's mean after every step, every push and pull
error buffer, every rank's outputs.  W in {2,3,4,5,7,8} covers the IEEE /W branch of
K5m (W not a power of two) and its shared memory sized for 8 sources; s in {1.0, 1.9};
gaussian (per-rank scales), block-sparse and all-zero gradients; reading R24 (a NaN in
one rank's push poisons that context's mean, every rank skips its pull).  Ref: P:182-187
(push, "servers average the gradients", pull), P:337-343 (shared compressed pull)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
f32 = np.float32

SIZES_SMALL = [432, 2304, 9216, 36864, 640, 60_001, 150_000]
SIZES_LARGE = [432, 2304, 9216, 36864, 640, 200_003, 1_000_000]
STEPS = 3


def _grads(r, step, sizes, kind):
    import synth

    if kind == "zeros":
        return [synth.zeros(n) for n in sizes]
    if kind == "sparse":
        def block_sparse(n, t):
            g = synth.gaussian(n, 95, r, t, step)
            j = np.arange(n) % -(-n // 5)
            g[(j // 10000) % 2 == 1] = 0.0
            return g

        return [synth.zeros(n) if t % 3 == 1 else block_sparse(n, t) if t % 3 == 0 else
                synth.gaussian(n, 95, r, t, step) for t, n in enumerate(sizes)]
    gs = [(synth.gaussian(n, 95, r, t, step) * f32(1.5 ** r)).astype(f32) for t, n in enumerate(sizes)]
    if kind == "nan" and step == 1 and r == 1:
        gs[5][7] = np.nan                      # one rank's push of one context fails (R24)
    return gs


def _run_group(W, sizes, s, kind, steps=STEPS, graph=False):
    import torch

    import paper_1802_07389_b200 as T

    dev = torch.device("cuda", torch.cuda.current_device())
    g = T.Loopback(W, sizes, dev)
    gs = [[torch.empty(n, device=dev) for n in sizes] for _ in range(W)]
    outs = [[torch.zeros(n, device=dev) for n in sizes] for _ in range(W)]
    owned, statuses = [], []
    gpush = gpull = None
    for step in range(steps):
        for r in range(W):
            for b, a in zip(gs[r], _grads(r, step, sizes, kind)):
                b.copy_(torch.from_numpy(a))
        if gpush is None:
            g.push(gs, s)
        else:
            gpush.replay()
        torch.cuda.synchronize()
        owned.append([x.owned.cpu().numpy().copy() for x in g.ranks])
        if gpull is None:
            g.pull(outs, s)                    # delta = mean (R18)
        else:
            gpull.replay()
        torch.cuda.synchronize()
        statuses.append([x.status() for x in g.ranks])
        if graph and gpush is None:
            gpush, gpull = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
            with torch.cuda.graph(gpush, capture_error_mode="thread_local"):
                g.push(gs, s)
            with torch.cuda.graph(gpull, capture_error_mode="thread_local"):
                g.pull(outs, s)
    res = [{"ctx": x.contexts(), "owned": [o[r] for o in owned], "outs": [o.cpu().numpy() for o in outs[r]],
            "push_err": x.push_err.cpu().numpy().copy(), "pull_err": x.pull_err.cpu().numpy().copy(),
            "status": [st[r] for st in statuses]} for r, x in enumerate(g.ranks)]
    g.close()
    return res


def _check(W, results, sizes, s, kind, steps=STEPS):
    from oracle import exchange as X

    ps = X.VirtualPS(sizes, W)
    outs = [[np.zeros(n, f32) for n in sizes] for _ in range(W)]
    means_steps, bad_steps = [], []
    for step in range(steps):
        means, sent = ps.push([_grads(r, step, sizes, kind) for r in range(W)], s)
        shared = ps.pull(means, outs, s)
        means_steps.append(means)
        bad_steps.append(any(p.status for p in shared))
    for r in range(W):
        res = results[r]
        for step in range(steps):
            assert (res["status"][step] != 0) == bad_steps[step], (r, step, res["status"][step])
            if bad_steps[step]:
                assert res["status"][step] == 2                     # TLC_ERR_NONFINITE on every rank
        for c, cx in enumerate(res["ctx"]):
            assert (cx["tensor"], cx["lo"], cx["hi"], cx["owner"]) == ps.ctx[c]
            n = cx["hi"] - cx["lo"]
            pe = res["push_err"][cx["elem_off"]: cx["elem_off"] + n]
            assert np.array_equal(pe.view(np.uint32), ps.push_err[r][c].view(np.uint32)), ("push_err", r, c)
            if cx["owner"] == r:
                for step in range(steps):
                    m = res["owned"][step][cx["owned_off"]: cx["owned_off"] + n]
                    ref = means_steps[step][c]
                    if np.isnan(ref).any():
                        assert np.isnan(m).all(), ("poisoned mean", r, c, step)
                    else:
                        assert np.array_equal(m.view(np.uint32), ref.view(np.uint32)), ("mean", r, c, step)
                pl = res["pull_err"][cx["owned_off"]: cx["owned_off"] + n]
                assert np.array_equal(pl.view(np.uint32), ps.pull_err[c].view(np.uint32)), ("pull_err", r, c)
        for t in range(len(sizes)):
            assert np.array_equal(res["outs"][t].view(np.uint32), outs[r][t].view(np.uint32)), ("out", r, t)


@pytest.mark.parametrize("kind", ["gauss", "sparse", "zeros"])
@pytest.mark.parametrize("s", [1.0, 1.9])
@pytest.mark.parametrize("W", [2, 3, 4, 5, 7, 8])
def test_loopback_matches_oracle(W, s, kind):
    _check(W, _run_group(W, SIZES_SMALL, s, kind), SIZES_SMALL, s, kind)


@pytest.mark.parametrize("W", [3, 8])
def test_loopback_large_contexts(W):
    """Contexts above the small-tensor bound: the streaming K1-K5 tables on both sides."""
    _check(W, _run_group(W, SIZES_LARGE, 1.75, "gauss"), SIZES_LARGE, 1.75, "gauss")


@pytest.mark.parametrize("W", [2, 3])
def test_loopback_producer_seeks_skip_k4(W):
    """Peer-memory consumers read the seek entries the producing K3 wrote (its phase 3 knows
    the payload offset and run carry at every K5 tile start) and launch no K4: the owners'
    K5m and every rank's apply still match the oracle bit for bit.  The contexts' last K3
    chunks are partial with K5 tile starts inside them (K3 gives every warp whole rows)."""
    import os

    import paper_1802_07389_b200 as T

    # W = 2: P = 28709 (its last 8 KiB chunk holds 4133 bytes, the tile start 28672 inside);
    # W = 3: two shards of P = 14355 (tile start 12288 inside a 6163-byte last chunk)
    sizes = [5 * (3 * 8192 + 4096 + 37), 5 * (4096 + 1) + 3, 40_961 * 3, 2304]
    T.tlc_prof_collect()
    T.tlc_prof_enable(True)
    try:
        res = _run_group(W, sizes, 1.5, "gauss", steps=2)
    finally:
        T.tlc_prof_enable(False)
    prof = T.tlc_prof_collect()
    _check(W, res, sizes, 1.5, "gauss", steps=2)
    k4 = prof.get("k4_zre_scan", (0, 0.0))[0]
    if os.environ.get("TLC_NO_PRODSEEK") == "1":
        assert k4 > 0, prof
    else:
        assert k4 == 0, prof
        assert prof.get("k3_zre", (0, 0.0))[0] > 0, prof


@pytest.mark.parametrize("W", [2, 4, 8])
def test_loopback_resnet110_small_tables(W):
    """BASELINE configs[3] (C4): ResNet-110's 110 layers -- every context is a small tensor, so
    the pushes and the owners' pulls are compressed by K6g (clusters) and the applies
    decompressed by K7 over records; owners' means, error buffers and outputs bit for bit."""
    import synth

    sizes = synth.RESNET110_SIZES
    _check(W, _run_group(W, sizes, 1.75, "gauss", steps=2), sizes, 1.75, "gauss", steps=2)


@pytest.mark.parametrize("W", [1, 5])
def test_loopback_graph_replay(W):
    _check(W, _run_group(W, SIZES_SMALL, 1.75, "gauss", graph=True), SIZES_SMALL, 1.75, "gauss")


@pytest.mark.parametrize("W", [2, 7])
def test_loopback_failed_push_poisons_context(W):
    """R24: rank 1's NaN at step 1 makes that context's mean NaN on its owner, the shared
    pull raises NONFINITE, every rank reports it and leaves that context untouched."""
    _check(W, _run_group(W, SIZES_SMALL, 1.5, "nan"), SIZES_SMALL, 1.5, "nan")


def test_loopback_phase_order_and_arguments():
    import torch

    import paper_1802_07389_b200 as T

    dev = torch.device("cuda", torch.cuda.current_device())
    g = T.Loopback(3, [1000, 70], dev)
    gs = [[torch.zeros(1000, device=dev), torch.zeros(70, device=dev)] for _ in range(3)]
    with pytest.raises(T.TlcError):
        g.pull(gs, 1.5)                                   # pull before push
    with pytest.raises(ValueError):
        g.push(gs[:2], 1.5)                               # a rank missing
    with pytest.raises(ValueError):
        g.push([[torch.zeros(999, device=dev), gs[r][1]] for r in range(3)], 1.5)
    g.push(gs, 1.5)
    with pytest.raises(T.TlcError):
        g.push(gs, 1.5)                                   # push twice
    g.pull(gs, 1.5)
    with pytest.raises(T.TlcError):
        g.ranks[0].push(gs[0], 1.5)                       # a virtual rank is driven by its group
    torch.cuda.synchronize()
    g.close()


def test_loopback_bert_large_full_size_sampled():
    """The bench's exchange workload at full size (BASELINE configs[4]: BERT-large, 150 tensors,
    335,869,952 values per rank, s = 1.9) with W = 4 virtual ranks, two steps: every rank's
    outputs bitwise identical (the shared pull), and for five sampled contexts (the largest, the
    smallest and three random) every rank's push error, the owner's mean, pull error and every
    rank's output equal to the oracle replaying those contexts alone (contexts are independent:
    X2-X6 per context)."""
    import torch

    import paper_1802_07389_b200 as T
    import synth
    from oracle import exchange as X

    W, s, steps = 4, 1.9, 2
    dev = torch.device("cuda", 0)
    sizes = synth.BERT_LARGE_SIZES
    g = T.Loopback(W, sizes, dev)
    ctxs = g.ranks[0].contexts()
    rng = np.random.default_rng(11)
    lens = [c["hi"] - c["lo"] for c in ctxs]
    pick = sorted({int(np.argmax(lens)), int(np.argmin(lens)), *rng.choice(len(ctxs), 3, replace=False).tolist()})
    sub = [(k, 0, lens[c], ctxs[c]["owner"]) for k, c in enumerate(pick)]
    ps = X.VirtualPS([lens[c] for c in pick], W, ctx=sub)
    outs = [[torch.zeros(n, device=dev) for n in sizes] for _ in range(W)]
    ref_outs = [[np.zeros(lens[c], f32) for c in pick] for _ in range(W)]
    for step in range(steps):
        grads = [synth.model_step_torch("bert-large", step, r, dev) for r in range(W)]
        g.push(grads, s)
        torch.cuda.synchronize()
        sub_grads = [[grads[r][ctxs[c]["tensor"]][ctxs[c]["lo"]:ctxs[c]["hi"]].cpu().numpy() for c in pick]
                     for r in range(W)]
        means, _ = ps.push(sub_grads, s)
        for k, c in enumerate(pick):
            o = ctxs[c]["owner"]
            oo = g.ranks[o].contexts()[c]["owned_off"]
            m = g.ranks[o].owned[oo: oo + lens[c]].cpu().numpy()
            assert np.array_equal(m.view(np.uint32), means[k].view(np.uint32)), ("mean", step, c)
        g.pull(outs, s)
        torch.cuda.synchronize()
        ps.pull(means, ref_outs, s)
        del grads
    for r in range(1, W):
        for t in range(len(sizes)):
            assert torch.equal(outs[r][t].view(torch.int32), outs[0][t].view(torch.int32)), (r, t)
    for k, c in enumerate(pick):
        cx = ctxs[c]
        for r in range(W):
            pe = g.ranks[r].push_err[cx["elem_off"]: cx["elem_off"] + lens[c]].cpu().numpy()
            assert np.array_equal(pe.view(np.uint32), ps.push_err[r][k].view(np.uint32)), ("push_err", r, c)
            o = outs[r][cx["tensor"]][cx["lo"]: cx["hi"]].cpu().numpy()
            assert np.array_equal(o.view(np.uint32), ref_outs[r][k].view(np.uint32)), ("out", r, c)
        own = g.ranks[cx["owner"]]
        oo = own.contexts()[c]["owned_off"]
        pl = own.pull_err[oo: oo + lens[c]].cpu().numpy()
        assert np.array_equal(pl.view(np.uint32), ps.pull_err[k].view(np.uint32)), ("pull_err", c)
    g.close()
