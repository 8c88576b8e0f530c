"""PyTorch DistributedDataParallel communication hook over the 3LC exchange
(the analog of the paper's distributed-optimizer integration,
P:576-594, with per-bucket exchanges as gradients become ready).

DDP hands the hook each gradient bucket (a flat fp32 tensor) as soon as backward
has produced it, so the compression of bucket k overlaps the backward pass of the
layers behind it.  Per bucket the hook runs the parameter-server step of
``Exchange`` (include/tlc.h): push -- compress with the bucket's push error
buffer, owners aggregate the W payloads into the mean -- and pull -- owners
compress the mean once with their pull error buffers, every rank decompresses
the deltas (skip-zero, R16) into a zeroed output.  The hook returns that output,
the same on every rank, as the bucket's reduced gradient.  All of it runs in the
library's kernels on the current stream; torch supplies the process group (id and
IPC-handle exchange at setup) and the bucket tensors.

    state = TLCHookState(s=1.75)
    ddp_model.register_comm_hook(state, tlc_hook)
"""
import torch
import torch.distributed as dist

from . import Comm, Exchange


class TLCHookState:
    """Hook state: the library communicator and one Exchange (with its error
    buffers) per DDP bucket, created on first use and rebuilt if DDP re-buckets."""

    def __init__(self, process_group=None, s: float = 1.75, use_zre: bool = True, p2p: bool = True):
        if not (1.0 <= s < 2.0):
            raise ValueError("s must be in [1, 2)")
        self.group = process_group
        self.rank = dist.get_rank(process_group)
        self.world = dist.get_world_size(process_group)
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.s, self.use_zre, self.p2p = float(s), bool(use_zre), bool(p2p)
        self.comm = Comm(self.rank, self.world, self.device, group=process_group)
        self.buckets = {}          # bucket index -> (numel, Exchange, output tensor)

    def exchange_for(self, index: int, numel: int):
        e = self.buckets.get(index)
        if e is None or e[0] != numel:
            if e is not None:
                e[1].close()
            x = Exchange(self.comm, [numel], p2p=self.p2p, group=self.group)
            e = (numel, x, torch.empty(numel, dtype=torch.float32, device=self.device))
            self.buckets[index] = e
        return e

    def close(self):
        for _, x, _ in self.buckets.values():
            x.close()
        self.buckets.clear()
        self.comm.close()


def tlc_hook(state: TLCHookState, bucket) -> torch.futures.Future[torch.Tensor]:
    """DDP comm hook: 3LC-compressed parameter-server exchange of one bucket."""
    grad = bucket.buffer()
    if grad.dtype != torch.float32 or not grad.is_cuda:
        raise TypeError("tlc_hook exchanges fp32 CUDA gradient buckets")
    grad = grad.contiguous()
    _, x, out = state.exchange_for(bucket.index(), grad.numel())
    stream = torch.cuda.current_stream()
    x.push([grad], state.s, state.use_zre, stream)
    out.zero_()
    x.pull([out], state.s, state.use_zre, stream)
    fut = torch.futures.Future()
    fut.set_result(out)
    return fut
