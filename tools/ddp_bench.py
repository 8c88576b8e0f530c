"""NEXT-2 measurement: one DDP training step (forward, backward with the gradient
exchange, SGD step) of an MLP with ~100M fp32 parameters, default NCCL all-reduce
vs the 3LC comm hook (paper_1802_07389_b200/ddp.py), max over ranks.

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/ddp_bench.py
"""
import json
import os
import sys

import torch
import torch.distributed as dist
from torch.nn.parallel import DistributedDataParallel as DDP

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_07389_b200.ddp import TLCHookState, tlc_hook  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    width, depth, batch, steps = 4096, 6, 64, 20
    res = {}
    for mode in ("allreduce", "tlc_p2p", "tlc_p2p_batch", "tlc_nccl"):
        torch.manual_seed(0)
        layers = []
        for _ in range(depth):
            layers += [torch.nn.Linear(width, width), torch.nn.ReLU()]
        model = torch.nn.Sequential(*layers).to(dev)
        ddp = DDP(model, device_ids=[local])
        state = None
        if mode != "allreduce":
            state = TLCHookState(s=1.75, p2p=mode.startswith("tlc_p2p"), batch=mode.endswith("batch"))
            ddp.register_comm_hook(state, tlc_hook)
        opt = torch.optim.SGD(ddp.parameters(), lr=1e-4)
        x = torch.randn(batch, width, device=dev)

        def step():
            opt.zero_grad(set_to_none=False)
            ddp(x).square().mean().backward()
            opt.step()

        for _ in range(5):
            step()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            step()
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / steps], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        res[mode] = float(t.item())
        if state is not None:
            state.close()
        del ddp, model, opt
        torch.cuda.empty_cache()
    nparam = depth * (width * width + width)
    if rank == 0:
        print(json.dumps({"what": "DDP step (fwd + bwd with gradient exchange + SGD) of a "
                                  f"{depth}x{width} MLP, {nparam:,} fp32 params, batch {batch}, {world} GPUs",
                          "ms_per_step": res, "params": nparam, "world": world}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
