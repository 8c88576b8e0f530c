"""The N>1 exchange protocol on CPU: 2 ranks over torch.distributed (gloo) run the
push/pull message pattern of csrc/exchange.cu (each owner receives every rank's
payload of its contexts; every rank receives every owner's shared pull payload)
with the oracle as the codec; every rank must end bit-identical to the
single-process W-virtual-rank oracle.  The product's plan is computed by
libtlc on each rank (host code, no GPU) and must agree across ranks."""
import os
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

f32 = np.float32
SIZES = [2304, 9216, 36864, 640, 432, 100_000]
S, STEPS = 1.5, 2


def _grads(r, step):
    import synth

    return [synth.gaussian(n, 91, r, t, step) for t, n in enumerate(SIZES)]


def _send_payload(p, dst):
    meta = torch.tensor([float(p.M), float(p.payload_len)], dtype=torch.float64)
    dist.send(meta, dst)
    if p.payload_len:
        dist.send(torch.from_numpy(p.payload.copy()), dst)


def _recv_payload(src):
    import oracle as O

    meta = torch.zeros(2, dtype=torch.float64)
    dist.recv(meta, src)
    ln = int(meta[1])
    buf = torch.zeros(ln, dtype=torch.uint8)
    if ln:
        dist.recv(buf, src)
    return O.Compressed(0, f32(meta[0]), 0, True, buf.numpy())


def _worker(rank, world, port, q):
    dist.init_process_group("gloo", init_method="file://" + port, rank=rank, world_size=world)
    try:
        import oracle as O
        import paper_1802_07389_b200 as T
        from oracle import exchange as X

        ctx = T.tlc_plan(SIZES, world)
        allplans = [None] * world
        dist.all_gather_object(allplans, ctx)
        assert all(p == ctx for p in allplans)
        assert ctx == X.plan(SIZES, world)
        push_err = [np.zeros(hi - lo, f32) for (_, lo, hi, _) in ctx]
        pull_err = {c: np.zeros(hi - lo, f32) for c, (_, lo, hi, o) in enumerate(ctx) if o == rank}
        outs = [np.zeros(n, f32) for n in SIZES]
        for step in range(STEPS):
            g = _grads(rank, step)
            sent = [O.compress(g[t][lo:hi], push_err[c], S) for c, (t, lo, hi, _) in enumerate(ctx)]
            # push: owners collect in rank order (sends/recvs ordered by context then rank)
            means = {}
            for c, (t, lo, hi, o) in enumerate(ctx):
                if o == rank:
                    got = []
                    for w in range(world):
                        got.append(sent[c] if w == rank else _recv_payload(w))
                    acc = np.zeros(hi - lo, f32)
                    for p in got:
                        st, acc = O.decompress(p.payload, True, p.M, hi - lo, out=acc, accumulate=True)
                    means[c] = (acc / f32(world)).astype(f32)
                else:
                    _send_payload(sent[c], o)
            # pull: each owner compresses once and sends to every other rank
            for c, (t, lo, hi, o) in enumerate(ctx):
                if o == rank:
                    p = O.compress(means[c], pull_err[c], S)
                    for w in range(world):
                        if w != rank:
                            _send_payload(p, w)
                else:
                    p = _recv_payload(o)
                view = outs[t][lo:hi].copy()
                st, view = O.decompress(p.payload, True, p.M, hi - lo, out=view, accumulate=True)
                outs[t][lo:hi] = view
        q.put((rank, [o.tobytes() for o in outs], [e.tobytes() for e in push_err],
               {c: e.tobytes() for c, e in pull_err.items()}))
    finally:
        dist.destroy_process_group()


def _free_port():
    # rendezvous through a file (FileStore): no port to race for with other processes
    p = os.path.join(tempfile.mkdtemp(prefix="tlc_rdv_"), "store")
    return p


def test_two_rank_gloo_protocol_matches_virtual_ps():
    from oracle import exchange as X

    world = 2
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    port = _free_port()
    procs = [ctxm.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict((r, (o, e, pe)) for r, o, e, pe in [q.get(timeout=300) for _ in range(world)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ps = X.VirtualPS(SIZES, world)
    outs = [[np.zeros(n, f32) for n in SIZES] for _ in range(world)]
    for step in range(STEPS):
        ps.step([_grads(r, step) for r in range(world)], outs, S)
    for r in range(world):
        o, e, pe = res[r]
        assert [x.tobytes() for x in outs[r]] == o
        assert [x.tobytes() for x in ps.push_err[r]] == e
        for c, b in pe.items():
            assert ps.pull_err[c].tobytes() == b
