"""NEXT-2: the DDP comm hook (paper_1802_07389_b200/ddp.py) on 2 GPUs.  Every bucket
the hook receives and returns is recorded; the returned reduced gradients must equal,
bit for bit, the W-virtual-rank oracle (oracle/exchange.py) run on the recorded
per-rank bucket gradients, step after step (error buffers carried per bucket)."""
import os
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
S, STEPS = 1.75, 4


def _worker(rank, world, port, q, p2p, batch=False, nan_step=-1):
    import torch
    import torch.distributed as dist
    from torch.nn.parallel import DistributedDataParallel as DDP

    from paper_1802_07389_b200.ddp import TLCHookState, tlc_hook

    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", init_method="file://" + port, rank=rank, world_size=world, device_id=dev)
    try:
        torch.manual_seed(0)
        model = torch.nn.Sequential(torch.nn.Linear(64, 256), torch.nn.ReLU(), torch.nn.Linear(256, 300),
                                    torch.nn.ReLU(), torch.nn.Linear(300, 10)).to(dev)
        ddp = DDP(model, device_ids=[rank], bucket_cap_mb=0.1)
        state = TLCHookState(s=S, p2p=p2p, batch=batch)
        steps = []

        def hook(st, bucket):
            inp = bucket.buffer().detach().clone()
            if rank == 1 and len(steps) - 1 == nan_step and bucket.index() == 0:   # steps[-1]: this step
                bucket.buffer()[3] = float("nan")           # one rank's gradient goes non-finite
                inp = bucket.buffer().detach().clone()
            fut = tlc_hook(st, bucket)
            steps[-1].append((bucket.index(), inp, fut))
            return fut

        ddp.register_comm_hook(state, hook)
        opt = torch.optim.SGD(ddp.parameters(), lr=0.01)
        g = torch.Generator(device="cpu").manual_seed(100 + rank)
        rec = []
        for step in range(STEPS):
            x = torch.randn(32, 64, generator=g).to(dev)
            opt.zero_grad()
            steps.append([])
            loss = ddp(x).square().mean()
            loss.backward()
            torch.cuda.synchronize()
            rec.append([(i, inp.cpu().numpy(), f.value().detach().clone().cpu().numpy()) for i, inp, f in steps[-1]])
            if step != nan_step:
                opt.step()
        params = [p.detach().cpu().numpy() for p in model.parameters()]
        q.put((rank, rec, params))
        state.close()
    finally:
        dist.destroy_process_group()


def _launch(world, p2p, batch=False, nan_step=-1):
    import torch.multiprocessing as mp

    # rendezvous through a file (FileStore): no port to race for with other processes
    port = os.path.join(tempfile.mkdtemp(prefix="tlc_rdv_"), "store")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, p2p, batch, nan_step)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict((r, (rec, params)) for r, rec, params in (q.get(timeout=600) for _ in range(world)))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


def _oracle_check(res, world, batch, nan_step=-1):
    from oracle import exchange as X

    rec0, rec1 = res[0][0], res[1][0]
    assert len(rec0) == len(rec1) == STEPS
    ps = {}
    for step, (b0s, b1s) in enumerate(zip(rec0, rec1)):
        assert [b[0] for b in b0s] == [b[0] for b in b1s]
        groups = [sorted(zip(b0s, b1s), key=lambda e: e[0][0])] if batch else [[e] for e in zip(b0s, b1s)]
        for grp in groups:
            sizes = tuple(a[1].size for a, _ in grp)
            key = sizes if batch else grp[0][0][0]
            if key not in ps or ps[key][0] != sizes:
                ps[key] = (sizes, X.VirtualPS(list(sizes), world))
            vp = ps[key][1]
            means, _ = vp.push([[a[1].astype(np.float32) for a, _ in grp], [b[1].astype(np.float32) for _, b in grp]], S)
            outs = [[np.zeros(n, np.float32) for n in sizes] for _ in range(world)]
            shared = vp.pull(means, outs, S)
            failed = any(p.status for p in shared)
            for k, (a, b) in enumerate(grp):
                if failed:                                   # R24: every rank gets NaN
                    assert np.isnan(a[2]).all() and np.isnan(b[2]).all(), (step, k)
                    continue
                assert np.array_equal(a[2].view(np.uint32), outs[0][k].view(np.uint32)), ("rank 0", step, a[0])
                assert np.array_equal(b[2].view(np.uint32), outs[1][k].view(np.uint32)), ("rank 1", step, b[0])
            if step == nan_step and grp[0][0][0] == 0:       # the bucket that got the NaN
                assert failed
    # identical reduced gradients -> identical (finite) parameters on both ranks
    for a, b in zip(res[0][1], res[1][1]):
        assert np.isfinite(a).all() and np.array_equal(a, b)


@pytest.mark.parametrize("p2p,batch", [(False, False), (True, False), (True, True)])
def test_ddp_hook_matches_oracle(p2p, batch):
    import torch

    world = 2
    if torch.cuda.device_count() < world:
        pytest.skip("needs 2 GPUs")
    _oracle_check(_launch(world, p2p, batch), world, batch)


@pytest.mark.parametrize("batch", [False, True])
def test_ddp_hook_nonfinite_gradient_is_nan_on_every_rank(batch):
    import torch

    world = 2
    if torch.cuda.device_count() < world:
        pytest.skip("needs 2 GPUs")
    _oracle_check(_launch(world, True, batch, nan_step=1), world, batch, nan_step=1)


@pytest.mark.parametrize("batch", [False, True])
def test_ddp_hook_world1_on_one_gpu(batch):
    """The hook's code path on one GPU (DDP with a world of 1, NCCL process group): every
    bucket's reduced gradient equals the oracle's W = 1 exchange of it (compress, decompress as
    the mean, shared pull), step after step with the error buffers carried; the batched schedule
    exchanges all buckets of a step together."""
    import torch.multiprocessing as mp

    # rendezvous through a file (FileStore): no port to race for with other processes
    port = os.path.join(tempfile.mkdtemp(prefix="tlc_rdv_"), "store")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_worker, args=(0, 1, port, q, True, batch, -1))
    p.start()
    r, rec, params = q.get(timeout=600)
    p.join(timeout=120)
    assert p.exitcode == 0
    from oracle import exchange as X

    assert len(rec) == STEPS
    ps = {}
    for step, bs in enumerate(rec):
        groups = [sorted(bs, key=lambda e: e[0])] if batch else [[e] for e in bs]
        for grp in groups:
            sizes = tuple(b[1].size for b in grp)
            key = sizes if batch else grp[0][0]
            if key not in ps or ps[key][0] != sizes:
                ps[key] = (sizes, X.VirtualPS(list(sizes), 1))
            vp = ps[key][1]
            means, _ = vp.push([[b[1].astype(np.float32) for b in grp]], S)
            outs = [[np.zeros(n, np.float32) for n in sizes]]
            vp.pull(means, outs, S)
            for k, b in enumerate(grp):
                assert np.array_equal(b[2].view(np.uint32), outs[0][k].view(np.uint32)), (step, b[0])
    assert all(np.isfinite(a).all() for a in params)
