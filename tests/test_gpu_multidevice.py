"""One process driving two GPUs: kernel attributes are per device (dynamic shared memory
limits of K2 bulk, K3, K6g, K7, K5m), the profiler's events are per device, and the fused
aggregate may read a peer GPU's payloads (peer access, NVLink).  Results bit for bit equal
to the single-device runs and to the oracle."""
import ctypes
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _peer(rt_dev_from, rt_dev_to):
    import torch

    path = "/usr/local/cuda/lib64/libcudart.so"
    rt = ctypes.CDLL(path if os.path.exists(path) else "libcudart.so.12")
    torch.cuda.set_device(rt_dev_from)
    rc = rt.cudaDeviceEnablePeerAccess(rt_dev_to, 0)
    assert rc in (0, 704), rc                       # 704: already enabled


@pytest.mark.parametrize("sizes", [[432, 2304, 9216, 36864, 640], [(1 << 22) + 3, 70_001, 1 << 20]])
def test_two_devices_one_process(sizes):
    import torch

    import oracle as O
    import paper_1802_07389_b200 as T
    import synth

    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    s = 1.75
    T.tlc_prof_enable(True)
    sets, grads = [], []
    for d in (0, 1):
        dev = torch.device("cuda", d)
        torch.cuda.set_device(dev)
        g = [synth.gaussian(n, 31, d, k) for k, n in enumerate(sizes)]
        ts = T.TensorSet(sizes, dev)
        ts.compress([torch.from_numpy(x).to(dev) for x in g], s, True)
        torch.cuda.synchronize(dev)
        sets.append(ts)
        grads.append(g)
    T.tlc_prof_collect()
    T.tlc_prof_enable(False)
    for d in (0, 1):
        hs = sets[d].headers()
        for k, n in enumerate(sizes):
            c = O.compress(grads[d][k], np.zeros(n, np.float32), s, True)
            assert hs[k]["status"] == 0 and hs[k]["payload_len"] == c.payload_len, (d, k)
            np.testing.assert_array_equal(sets[d].payloads[k][: c.payload_len].cpu().numpy(), c.payload)
    # the mean on cuda:0 with source 1 read from cuda:1 (peer memory) == with source 1 copied over
    _peer(0, 1)
    d0 = torch.device("cuda", 0)
    outs = [torch.empty(n, device=d0) for n in sizes]
    T.Aggregate(outs, [(sets[0].payloads, sets[0].hdrs), (sets[1].payloads, sets[1].hdrs)]).run()
    outs_l = [torch.empty(n, device=d0) for n in sizes]
    T.Aggregate(outs_l, [(sets[0].payloads, sets[0].hdrs), ([p.to(d0) for p in sets[1].payloads], sets[1].hdrs.to(d0))]).run()
    torch.cuda.synchronize(d0)
    for a, b in zip(outs, outs_l):
        assert torch.equal(a.view(torch.int32), b.view(torch.int32))
