"""NEXT-2: the DDP comm hook (paper_1802_07389_b200/ddp.py) on 2 GPUs.  Every bucket
the hook receives and returns is recorded; the returned reduced gradients must equal,
bit for bit, the W-virtual-rank oracle (oracle/exchange.py) run on the recorded
per-rank bucket gradients, step after step (error buffers carried per bucket)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
S, STEPS = 1.75, 4


def _worker(rank, world, port, q, p2p):
    import torch
    import torch.distributed as dist
    from torch.nn.parallel import DistributedDataParallel as DDP

    from paper_1802_07389_b200.ddp import TLCHookState, tlc_hook

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    try:
        torch.manual_seed(0)
        model = torch.nn.Sequential(torch.nn.Linear(64, 256), torch.nn.ReLU(), torch.nn.Linear(256, 300),
                                    torch.nn.ReLU(), torch.nn.Linear(300, 10)).to(dev)
        ddp = DDP(model, device_ids=[rank], bucket_cap_mb=0.1)
        state = TLCHookState(s=S, p2p=p2p)
        rec = []

        def hook(st, bucket):
            inp = bucket.buffer().detach().clone()
            fut = tlc_hook(st, bucket)
            rec.append((len(rec), bucket.index(), inp.cpu().numpy(), fut.value().detach().clone().cpu().numpy()))
            return fut

        ddp.register_comm_hook(state, hook)
        opt = torch.optim.SGD(ddp.parameters(), lr=0.01)
        g = torch.Generator(device="cpu").manual_seed(100 + rank)
        grads_ok = True
        for step in range(STEPS):
            x = torch.randn(32, 64, generator=g).to(dev)
            opt.zero_grad()
            loss = ddp(x).square().mean()
            loss.backward()
            torch.cuda.synchronize()
            opt.step()
        params = [p.detach().cpu().numpy() for p in model.parameters()]
        q.put((rank, rec, params, grads_ok))
        state.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("p2p", [False, True])
def test_ddp_hook_matches_oracle(p2p):
    import torch
    import torch.multiprocessing as mp

    from oracle import exchange as X

    world = 2
    if torch.cuda.device_count() < world:
        pytest.skip("needs 2 GPUs")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, p2p)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict((r, (rec, params)) for r, rec, params, _ in (q.get(timeout=600) for _ in range(world)))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    rec0, rec1 = res[0][0], res[1][0]
    assert len(rec0) == len(rec1) and len(rec0) >= STEPS
    ps = {}
    for (i0, b0, in0, out0), (i1, b1, in1, out1) in zip(rec0, rec1):
        assert b0 == b1 and in0.size == in1.size
        key = b0
        if key not in ps or ps[key][0] != in0.size:
            ps[key] = (in0.size, X.VirtualPS([in0.size], world))
        vp = ps[key][1]
        means, _ = vp.push([[in0.astype(np.float32)], [in1.astype(np.float32)]], S)
        outs = [[np.zeros(in0.size, np.float32)] for _ in range(world)]
        vp.pull(means, outs, S)
        assert np.array_equal(out0.view(np.uint32), outs[0][0].view(np.uint32)), ("rank 0", i0, b0)
        assert np.array_equal(out1.view(np.uint32), outs[1][0].view(np.uint32)), ("rank 1", i1, b1)
    # identical reduced gradients -> identical parameters on both ranks
    for a, b in zip(res[0][1], res[1][1]):
        assert np.array_equal(a, b)
