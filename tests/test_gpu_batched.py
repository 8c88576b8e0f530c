"""Batches of tensors (tlc_batch_*, segment tables through K1-K5) vs the CPU
oracle, tensor by tensor, bit for bit (BASELINE configs[1]: ResNet-110)."""
import numpy as np
import pytest

import oracle as O
import synth

pytestmark = pytest.mark.gpu
f32 = np.float32


@pytest.fixture(scope="module")
def T():
    import torch

    assert torch.cuda.is_available()
    import paper_1802_07389_b200 as T

    return T


def _run_steps(T, sizes, steps, s, use_zre, make_t):
    import torch

    ts_set = T.TensorSet(sizes)
    bufs = [np.zeros(n, f32) for n in sizes]
    for step in range(steps):
        tl = [make_t(k, n, step) for k, n in enumerate(sizes)]
        td = [torch.from_numpy(x).cuda() for x in tl]
        ts_set.compress(td, s, use_zre)
        outs = [torch.full((n,), float("nan"), device="cuda") for n in sizes]
        accs = [torch.from_numpy(synth.gaussian(n, 77, k)).cuda() for k, n in enumerate(sizes)]
        acc0 = [a.cpu().numpy().copy() for a in accs]
        ts_set.decompress(outs)
        ts_set.decompress(accs, mode=T.TLC_MODE_ACCUMULATE)
        torch.cuda.synchronize()
        hs = ts_set.headers()
        for k, n in enumerate(sizes):
            c = O.compress(tl[k], bufs[k], s, use_zre)
            h = hs[k]
            assert h["status"] == c.status, (k, n)
            if c.status != O.OK:
                continue
            assert np.float32(h["M"]) == c.M and h["payload_len"] == c.payload_len, (k, n, step)
            np.testing.assert_array_equal(ts_set.payloads[k][: c.payload_len].cpu().numpy(), c.payload)
            assert np.array_equal(ts_set.errs[k].cpu().numpy().view(np.uint32), bufs[k].view(np.uint32))
            st, ref = O.decompress(c.payload, use_zre, c.M, n)
            assert np.array_equal(outs[k].cpu().numpy().view(np.uint32), ref.view(np.uint32)), (k, n)
            st, refa = O.decompress(c.payload, use_zre, c.M, n, out=acc0[k].copy(), accumulate=True)
            assert np.array_equal(accs[k].cpu().numpy().view(np.uint32), refa.view(np.uint32)), (k, n)
    return ts_set


@pytest.mark.parametrize("s", [1.0, 1.75, 1.9])
def test_resnet110_batched(T, s):
    sizes = synth.RESNET110_SIZES
    mus = synth.layer_means(sizes, 2, 110)
    _run_steps(T, sizes, 3, s, True, lambda k, n, step: synth.layer_gradient(n, mus[k], 2, 0, k, step))


# small tables (every n <= 40,960): K6g cuts a tensor of r ZRE rows (1 KiB of quartic bytes
# each) into min(4, ceil(r/2)) slices -- these sizes give groups of 1, 2, 3 and 4 slices with
# uneven last rows, packed together into clusters of 4 -- and K7 takes 2048-position parts
SMALL_GROUP_SIZES = [1, 2, 7, 432, 5120, 5121, 10240, 10241, 15361, 20481, 30721, 40960, 36864,
                     9216, 2304, 640, 4608, 18432, 25603, 35839]


@pytest.mark.parametrize("use_zre", [True, False])
@pytest.mark.parametrize("s", [1.0, 1.9])
def test_small_table_group_shapes(T, s, use_zre):
    _run_steps(T, SMALL_GROUP_SIZES, 2, s, use_zre, lambda k, n, step: synth.runs_adversarial(n, 1.0, 9, k, step)
               if k % 3 == 0 else synth.gaussian(n, 9, k, step))


def test_mixed_sizes(T):
    sizes = list(range(1, 12)) + [69, 70, 71, 1000, 5 * 2048 + 3, 163_840, 163_841, 400_003, 5 * 65536 + 7]
    for use_zre in (True, False):
        _run_steps(T, sizes, 2, 1.5, use_zre, lambda k, n, step: synth.runs_adversarial(n, 1.0, 5, k, step)
                   if k % 2 else synth.gaussian(n, 6, k, step))


def test_nonfinite_tensor_in_batch(T):
    sizes = [5000, 6000, 7000]

    def make(k, n, step):
        x = synth.gaussian(n, 8, k, step)
        if k == 1:
            x[17] = np.nan
        return x

    ts = _run_steps(T, sizes, 1, 1.0, True, make)
    hs = ts.headers()
    assert [h["status"] for h in hs] == [0, 2, 0]


def test_batched_format_error_writes_nothing(T):
    import torch

    sizes = [7000, 7000]
    ts = T.TensorSet(sizes)
    td = [torch.from_numpy(synth.gaussian(n, 9, k)).cuda() for k, n in enumerate(sizes)]
    ts.compress(td, 1.0, True)
    torch.cuda.synchronize()
    b0 = int(ts.payloads[1][0])
    ts.payloads[1][0] = 243 if b0 == 255 else 255   # change the expansion length of tensor 1
    outs = [torch.full((n,), 7.0, device="cuda") for n in sizes]
    ts.decompress(outs)
    torch.cuda.synchronize()
    hs = ts.headers()
    assert hs[0]["status"] == 0 and hs[1]["status"] == T.TLC_ERR_FORMAT
    assert torch.all(outs[1] == 7.0)


@pytest.mark.parametrize("use_zre", [True, False])
def test_large_table_bulk_path(T, use_zre):
    """A table of >= 32M values (large work items, like BERT-large's): its complete K2 tiles go
    through the table form of the bulk-copy kernel, the rest through the register kernel;
    partitions of every alignment (P mod 4 = 0..3), a tiny tensor, two error-feedback steps."""
    sizes = [(1 << 24) + 3, (1 << 23) + 1, 1 << 22, (1 << 22) + 10, 1000, 70_001, (1 << 21) + 15]
    assert sum(sizes) >= 32 << 20
    _run_steps(T, sizes, 2, 1.75, use_zre, lambda k, n, step: synth.gaussian(n, 10, k, step))
