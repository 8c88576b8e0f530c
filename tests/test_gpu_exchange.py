"""The NCCL exchange (tlc_exchange_push / tlc_exchange_pull) vs the W-virtual-rank
oracle (oracle/exchange.py, X1-X6): owners' means, every rank's outputs and every
push / pull error buffer, bit for bit, eagerly and (peer-memory transport) replayed
from CUDA graphs.  W = 1 runs in-process; W = 2, 4 spawn one process per GPU when the
box has them."""
import os
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
f32 = np.float32

SIZES = [432, 2304, 9216, 36864, 640, 200_003, 1_000_000]
S, STEPS = 1.75, 3


def _grads(r, step, sizes=SIZES, kind="gauss"):
    import synth

    if kind == "sparse":
        # zero tiles next to nonzero ones in every payload: runs of zero groups crossing
        # decoder tiles, an all-zero tensor, and a gaussian one (owners skip zero windows)
        def block_sparse(n, t):
            g = synth.gaussian(n, 95, r, t, step)
            j = np.arange(n) % -(-n // 5)              # quartic position of each element
            g[(j // 10000) % 2 == 1] = 0.0              # zero groups in blocks over two tiles wide
            return g

        return [synth.zeros(n) if t % 3 == 1 else block_sparse(n, t) if t % 3 == 0 else
                synth.gaussian(n, 95, r, t, step) for t, n in enumerate(sizes)]
    return [synth.gaussian(n, 95, r, t, step) for t, n in enumerate(sizes)]


def _run_rank(rank, world, steps, sizes=SIZES, p2p=False, graph=False, kind="gauss", exact=False):
    """One rank's exchange; returns per-step means (owned flat) and final state.
    graph=True: step 0 runs eagerly (it uploads the descriptor tables), then push and
    pull are captured once as CUDA graphs over fixed gradient buffers and replayed."""
    import torch

    import paper_1802_07389_b200 as T

    dev = torch.device("cuda", torch.cuda.current_device())
    comm = T.Comm(rank, world, dev)
    x = T.Exchange(comm, sizes, p2p=p2p, exact=exact)
    outs = [torch.zeros(n, device=dev) for n in sizes]
    gs = [torch.empty(n, device=dev) for n in sizes]
    owned_per_step = []
    gpush = gpull = None
    for step in range(steps):
        for b, a in zip(gs, _grads(rank, step, sizes, kind)):
            b.copy_(torch.from_numpy(a))
        if gpush is None:
            x.push(gs, S)
        else:
            gpush.replay()
        torch.cuda.synchronize()
        owned_per_step.append(x.owned.cpu().numpy().copy())
        if gpull is None:
            x.pull(outs, S)      # delta = mean (R18)
        else:
            gpull.replay()
        torch.cuda.synchronize()
        if graph and gpush is None:
            gpush, gpull = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
            with torch.cuda.graph(gpush, capture_error_mode="thread_local"):
                x.push(gs, S)
            with torch.cuda.graph(gpull, capture_error_mode="thread_local"):
                x.pull(outs, S)
    assert x.status() == 0
    res = {"ctx": x.contexts(), "owned": owned_per_step, "outs": [o.cpu().numpy() for o in outs],
           "push_err": x.push_err.cpu().numpy().copy(), "pull_err": x.pull_err.cpu().numpy().copy()}
    x.close()
    comm.close()
    return res


def _check(world, results, sizes=SIZES, steps=STEPS, kind="gauss"):
    from oracle import exchange as X

    ps = X.VirtualPS(sizes, world)
    outs = [[np.zeros(n, f32) for n in sizes] for _ in range(world)]
    means_steps = []
    for step in range(steps):
        means, _ = ps.push([_grads(r, step, sizes, kind) for r in range(world)], S)
        ps.pull(means, outs, S)
        means_steps.append(means)
    for r in range(world):
        res = results[r]
        for c, cx in enumerate(res["ctx"]):
            assert (cx["tensor"], cx["lo"], cx["hi"], cx["owner"]) == ps.ctx[c]
            n = cx["hi"] - cx["lo"]
            pe = res["push_err"][cx["elem_off"]: cx["elem_off"] + n]
            assert np.array_equal(pe.view(np.uint32), ps.push_err[r][c].view(np.uint32)), ("push_err", r, c)
            if cx["owner"] == r:
                for step in range(steps):
                    m = res["owned"][step][cx["owned_off"]: cx["owned_off"] + n]
                    assert np.array_equal(m.view(np.uint32), means_steps[step][c].view(np.uint32)), ("mean", r, c)
                pl = res["pull_err"][cx["owned_off"]: cx["owned_off"] + n]
                assert np.array_equal(pl.view(np.uint32), ps.pull_err[c].view(np.uint32)), ("pull_err", r, c)
        for t in range(len(sizes)):
            assert np.array_equal(res["outs"][t].view(np.uint32), outs[r][t].view(np.uint32)), ("out", r, t)


@pytest.mark.parametrize("p2p,graph,exact", [(False, False, False), (False, False, True), (True, False, False),
                                            (True, True, False)])
def test_exchange_w1_in_process(p2p, graph, exact):
    import torch

    assert torch.cuda.is_available()
    _check(1, [_run_rank(0, 1, STEPS, p2p=p2p, graph=graph, exact=exact)])


def test_exchange_w1_sparse_gradients():
    """Payloads with all-zero decoder tiles between nonzero ones (the owners' aggregate and
    the pull's skip-zero apply skip those tiles' expansion), W = 1 in process."""
    _check(1, [_run_rank(0, 1, STEPS, p2p=True, kind="sparse")], kind="sparse")


def _mp_worker(rank, world, port, q, p2p, graph=False, kind="gauss", exact=False):
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", init_method="file://" + port, rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    try:
        res = _run_rank(rank, world, STEPS, p2p=p2p, graph=graph, kind=kind, exact=exact)
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("p2p,graph,kind,exact", [(False, False, "gauss", False), (False, False, "sparse", True),
                                                  (True, False, "gauss", False), (True, True, "gauss", False),
                                                  (True, False, "sparse", False)])
@pytest.mark.parametrize("world", [2, 4])
def test_exchange_multi_gpu(world, p2p, graph, kind, exact):
    import torch
    import torch.multiprocessing as mp

    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    # rendezvous through a file (FileStore): no port to race for with other processes
    port = os.path.join(tempfile.mkdtemp(prefix="tlc_rdv_"), "store")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_mp_worker, args=(r, world, port, q, p2p, graph, kind, exact)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    _check(world, results, kind=kind)


def test_nccl_transport_refuses_capture():
    """The NCCL transport returns TLC_ERR_ARG on a capturing stream (no hang)."""
    import torch

    import paper_1802_07389_b200 as T

    dev = torch.device("cuda", torch.cuda.current_device())
    comm = T.Comm(0, 1, dev)
    x = T.Exchange(comm, SIZES, p2p=False)
    gs = [torch.zeros(n, device=dev) for n in SIZES]
    x.push(gs, S)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with pytest.raises(T.TlcError):
        with torch.cuda.graph(g, capture_error_mode="thread_local"):
            x.push(gs, S)
    torch.cuda.synchronize()
    x.close()
    comm.close()
