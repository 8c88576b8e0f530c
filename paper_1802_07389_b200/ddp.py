"""PyTorch DistributedDataParallel communication hook over the 3LC exchange
(the analog of the paper's distributed-optimizer integration,
P:576-594, with per-bucket exchanges as gradients become ready).

DDP hands the hook each gradient bucket (a flat fp32 tensor) as soon as backward
has produced it.  Per bucket the hook runs the parameter-server step of
``Exchange`` (include/tlc.h): push -- compress with the bucket's push error
buffer, owners aggregate the W payloads into the mean -- and pull -- owners
compress the mean once with their pull error buffers, every rank decompresses
the deltas (skip-zero, R16) into a zeroed output.  The hook returns that output,
the same on every rank, as the bucket's reduced gradient.  All of it runs in the
library's kernels on the current stream; torch supplies the process group (id and
IPC-handle exchange at setup) and the bucket tensors.

Two schedules:
  * per bucket (default): bucket k's exchange is issued as soon as DDP hands it
    over, so it overlaps the backward of the layers behind it; one
    Exchange, two barriers and ~10 launches per bucket.
  * batch=True: the buckets of a step are collected and exchanged together when
    DDP hands over the last one (``bucket.is_last()``): one Exchange over all
    buckets, one push + one pull per step, no overlap with backward.

Failures (reading R24): if any rank's push of a bucket region is non-finite, the
exchange's status is NONFINITE on every rank; the hook then fills the returned
gradient with NaN, as an all-reduce of a NaN gradient would, so GradScaler and
anomaly detection see it (on the device: no host synchronization).

    state = TLCHookState(s=1.75)
    ddp_model.register_comm_hook(state, tlc_hook)
"""
import torch
import torch.distributed as dist

from . import Comm, Exchange


class TLCHookState:
    """Hook state: the library communicator and the Exchanges (with their error
    buffers), created on first use and rebuilt if DDP re-buckets."""

    def __init__(self, process_group=None, s: float = 1.75, use_zre: bool = True, p2p: bool = True,
                 batch: bool = False):
        if not (1.0 <= s < 2.0):
            raise ValueError("s must be in [1, 2)")
        self.group = process_group
        self.rank = dist.get_rank(process_group)
        self.world = dist.get_world_size(process_group)
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.s, self.use_zre, self.p2p, self.batch = float(s), bool(use_zre), bool(p2p), bool(batch)
        self.comm = Comm(self.rank, self.world, self.device, group=process_group)
        self.buckets = {}          # per-bucket schedule: index -> (numel, Exchange, output tensor)
        self.batched = {}          # batch schedule: tuple of bucket sizes -> (Exchange, outputs)
        self.pending = []          # batch schedule: (index, buffer, future) of this step
        self.status = torch.zeros(1, dtype=torch.int32, device=self.device)

    def exchange_for(self, index: int, numel: int):
        e = self.buckets.get(index)
        if e is None or e[0] != numel:
            if e is not None:
                e[1].close()
            x = Exchange(self.comm, [numel], p2p=self.p2p, group=self.group)
            e = (numel, x, torch.empty(numel, dtype=torch.float32, device=self.device))
            self.buckets[index] = e
        return e

    def batched_for(self, sizes):
        key = tuple(sizes)
        e = self.batched.get(key)
        if e is None:
            for x, _ in self.batched.values():
                x.close()
            self.batched.clear()
            x = Exchange(self.comm, list(sizes), p2p=self.p2p, group=self.group)
            e = (x, [torch.empty(n, dtype=torch.float32, device=self.device) for n in sizes])
            self.batched[key] = e
        return e

    def close(self):
        for _, x, _ in self.buckets.values():
            x.close()
        for x, _ in self.batched.values():
            x.close()
        self.buckets.clear()
        self.batched.clear()
        self.comm.close()


def _exchange(state: TLCHookState, x: Exchange, grads, outs, stream):
    x.push(grads, state.s, state.use_zre, stream)
    for o in outs:
        o.zero_()
    x.pull(outs, state.s, state.use_zre, stream)
    # R24: a failed push anywhere makes the step's status non-OK on every rank; poison the
    # reduced gradients (device-side, no host sync) instead of returning a finite bias
    x.status_async(state.status, stream)
    bad = state.status != 0
    for o in outs:
        o.masked_fill_(bad, float("nan"))


def tlc_hook(state: TLCHookState, bucket) -> torch.futures.Future[torch.Tensor]:
    """DDP comm hook: 3LC-compressed parameter-server exchange of one bucket (or, with
    batch=True, of all buckets of the step once the last one is ready)."""
    grad = bucket.buffer()
    if grad.dtype != torch.float32 or not grad.is_cuda:
        raise TypeError("tlc_hook exchanges fp32 CUDA gradient buckets")
    grad = grad.contiguous()
    stream = torch.cuda.current_stream()
    fut = torch.futures.Future()
    if not state.batch:
        _, x, out = state.exchange_for(bucket.index(), grad.numel())
        _exchange(state, x, [grad], [out], stream)
        fut.set_result(out)
        return fut
    state.pending.append((bucket.index(), grad, fut))
    if bucket.is_last():
        items = sorted(state.pending, key=lambda e: e[0])
        state.pending = []
        x, outs = state.batched_for([g.numel() for _, g, _ in items])
        _exchange(state, x, [g for _, g, _ in items], outs, stream)
        for (_, _, f), o in zip(items, outs):
            f.set_result(o)
    return fut
