"""Desk-scale data-parallel training simulator on one GPU (SPEC psim,
S:424-515): W virtual workers and one parameter server run the paper's BSP step (P:177-188,
fig. push-and-pull) with per-tensor compression contexts in both directions and a shared
compressed pull, so the codec's bits per state change can be watched over
training -- the trend of Table 2 and the push/pull shape of Fig. size-sm
 -- without CIFAR-10.

Step:
  1. every worker computes minibatch gradients of a 1-hidden-layer MLP on its shard of a
     synthetic Gaussian-blob task (synth.blobs) against its model replica;
  2. push: every worker compresses each compressed tensor (ndim >= 2, R19; biases go
     uncompressed) with its own push context;
  3. the server averages: the library's fused aggregation (tlc_aggregate: K4 + K5m) folds
     the W payloads in worker order from +0 and divides by W (R15, R16); the compared
     designs decompress-accumulate in worker order, uncompressed tensors are summed in
     worker order, then / W (IEEE, in torch);
  4. the server applies momentum SGD (0.9, cosine learning-rate decay) to the
     global model; the model delta is the update (R18);
  5. pull: the server compresses each delta ONCE with its pull context; every worker
     applies the same payload to its replica (skip-zero accumulate, R16).  Under BSP all
     replicas stay bit-identical, so one replica tensor stands for all W.

Codecs: "3lc" (tlc_batch compress / decompress; s, use_zre), "stoch" (Stoch 3-value + QE,
tlc_stoch_compress), "int8" (8-bit int), "none" (32-bit float).
Every compression, decompression and 3LC / Stoch aggregation (fold and / W) runs in libtlc's
kernels (the 8-bit and fp32 baselines' / W is a torch division); torch supplies
the model's forward/backward, the optimizer arithmetic and device memory.
"""
from __future__ import annotations

import dataclasses
import math

import torch

from . import (TLC_MODE_ACCUMULATE, Aggregate, TensorSet, new_header, parse_header, tlc_decompress, tlc_int8_compress,
               tlc_int8_decompress, tlc_int8_workspace_bytes, tlc_max_payload_bytes, tlc_stoch_compress,
               workspace)


@dataclasses.dataclass
class SimConfig:
    workers: int = 4
    steps: int = 300
    batch_per_worker: int = 32
    base_lr: float = 0.1
    cosine: bool = True
    momentum: float = 0.9
    codec: str = "3lc"               # 3lc | stoch | int8 | none
    s: float = 1.0
    use_zre: bool = True
    seed: int = 7
    input_dim: int = 64
    hidden: int = 256
    classes: int = 10
    n_train: int = 8192
    n_test: int = 2048
    blob_std: float = 0.7
    eval_every: int = 50


class Sim:
    def __init__(self, cfg: SimConfig, device=None):
        import synth

        self.cfg = c = cfg
        self.dev = dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        xtr, ytr, xte, yte = synth.blobs(c.n_train, c.n_test, c.input_dim, c.classes, c.blob_std, c.seed, 1)
        self.xtr, self.ytr = torch.from_numpy(xtr).to(dev), torch.from_numpy(ytr).to(dev)
        self.xte, self.yte = torch.from_numpy(xte).to(dev), torch.from_numpy(yte).to(dev)
        g = torch.Generator(device="cpu").manual_seed(c.seed)
        shapes = [(c.hidden, c.input_dim), (c.hidden,), (c.classes, c.hidden), (c.classes,)]
        fan = [c.input_dim, c.input_dim, c.hidden, c.hidden]
        self.global_params = [((torch.rand(sh, generator=g) * 2 - 1) / math.sqrt(f)).to(dev)
                              for sh, f in zip(shapes, fan)]
        self.replica = [p.clone() for p in self.global_params]      # every worker's model (BSP)
        self.velocity = [torch.zeros_like(p) for p in self.global_params]
        self.comp = [i for i, p in enumerate(self.global_params) if p.dim() >= 2]      # R19
        self.plain = [i for i in range(len(shapes)) if i not in self.comp]
        self.sizes = [self.global_params[i].numel() for i in self.comp]
        W = c.workers
        if c.codec == "3lc":
            self.push_ctx = [TensorSet(self.sizes, dev) for _ in range(W)]
            # the server's aggregation: the library's fused fold + / W over the W push payloads
            self.means = [torch.empty(n, dtype=torch.float32, device=dev) for n in self.sizes]
            self.agg = Aggregate(self.means, [(x.payloads, x.hdrs) for x in self.push_ctx])
        elif c.codec == "stoch":
            self.push_pay = [[torch.empty(max(1, tlc_max_payload_bytes(n)), dtype=torch.uint8, device=dev)
                              for n in self.sizes] for _ in range(W)]
            self.push_hdr = [[new_header(dev) for _ in self.sizes] for _ in range(W)]
            # Stoch 3-value + QE payloads decode like 3LC's (M = m): the same fused aggregation
            self.means = [torch.empty(n, dtype=torch.float32, device=dev) for n in self.sizes]
            self.agg = Aggregate(self.means, list(zip(self.push_pay, self.push_hdr)))
        elif c.codec == "int8":
            self.push_codes = [[torch.empty(n, dtype=torch.int8, device=dev) for n in self.sizes] for _ in range(W)]
            self.push_hdr = [[new_header(dev) for _ in self.sizes] for _ in range(W)]
        elif c.codec != "none":
            raise ValueError(c.codec)
        if c.codec in ("3lc", "stoch"):
            # the server's pull contexts: error buffers for 3LC; for the stochastic design (no
            # error buffer) only the payload / header storage of its pulls is used
            self.pull_ctx = TensorSet(self.sizes, dev)
        self.step_no = 0
        self.log = []
        self.order = torch.randperm(c.n_train, generator=g).to(dev)

    # ------------------------------------------------------------------ pieces
    def lr(self) -> float:
        c = self.cfg
        if not c.cosine:
            return c.base_lr
        f = min(1.0, self.step_no / max(1, c.steps))
        return 0.001 + 0.5 * (c.base_lr - 0.001) * (1 + math.cos(math.pi * f))   # 0.1 -> 0.001

    def _grads(self, w: int):
        c = self.cfg
        per = c.n_train // c.workers                 # contiguous equal shards
        k = (self.step_no * c.batch_per_worker) % max(1, per - c.batch_per_worker + 1)
        idx = self.order[w * per + k: w * per + k + c.batch_per_worker]
        x, y = self.xtr[idx], self.ytr[idx]
        ps = [p.detach().clone().requires_grad_(True) for p in self.replica]
        h = torch.relu(x @ ps[0].t() + ps[1])
        loss = torch.nn.functional.cross_entropy(h @ ps[2].t() + ps[3], y)
        loss.backward()
        return [p.grad.detach().contiguous().reshape(-1) for p in ps], float(loss.detach())

    def evaluate(self) -> float:
        p = self.global_params
        with torch.no_grad():
            logits = torch.relu(self.xte @ p[0].t() + p[1]) @ p[2].t() + p[3]
            return float((logits.argmax(1) == self.yte).float().mean())

    # ------------------------------------------------------------------ one BSP step
    def step(self, record: bool = False):
        c, W, dev = self.cfg, self.cfg.workers, self.dev
        grads, losses = zip(*[self._grads(w) for w in range(W)])
        if not all(map(math.isfinite, losses)):
            raise FloatingPointError(f"diverged at step {self.step_no}")
        sums = [torch.zeros(n, dtype=torch.float32, device=dev) for n in self.sizes]     # +0 (R15)
        push_bytes = 0
        for w in range(W):                                                             # worker order
            gw = [grads[w][i] for i in self.comp]
            if c.codec == "3lc":
                ctx = self.push_ctx[w]
                ctx.compress(gw, c.s, c.use_zre)
                hs = ctx.headers()
                push_bytes += sum(h["payload_len"] for h in hs)
            elif c.codec == "stoch":
                for k, g in enumerate(gw):
                    seed = (c.seed << 20) ^ (w << 8) ^ k
                    tlc_stoch_compress(g, seed, self.step_no, c.use_zre, self.push_pay[w][k], self.push_hdr[w][k])
                push_bytes += sum(parse_header(h)["payload_len"] for h in self.push_hdr[w])
            elif c.codec == "int8":
                for k, g in enumerate(gw):
                    tlc_int8_compress(g, self.push_codes[w][k], self.push_hdr[w][k],
                                      workspace(tlc_int8_workspace_bytes(g.numel()), dev, "int8"))
                    tlc_int8_decompress(self.push_codes[w][k], self.push_hdr[w][k], g.numel(), sums[k],
                                        TLC_MODE_ACCUMULATE)
                push_bytes += sum(g.numel() for g in gw)
            else:
                for k, g in enumerate(gw):
                    sums[k] += g
                push_bytes += 4 * sum(g.numel() for g in gw)
        if c.codec in ("3lc", "stoch"):
            # R15 in the library: rank-ordered fold from +0 of the nonzero trits, then the IEEE / W
            self.agg.run()
            means = [m.clone() for m in self.means]
        else:
            # 8-bit int / 32-bit float were summed into sums above in worker order; / W as an
            # IEEE fp32 division: an elementwise tensor divisor -- torch turns division by a
            # Python scalar into multiplication by its reciprocal, which differs for W = 3, 5, ...
            means = [torch.div(s, torch.full_like(s, float(W))) for s in sums]
        plain_means = []
        for i in self.plain:
            acc = torch.zeros_like(grads[0][i])
            for w in range(W):
                acc += grads[w][i]
            plain_means.append(torch.div(acc, torch.full_like(acc, float(W))))
        # server: momentum SGD on the global model; the delta is the update (R18)
        lr = self.lr()
        full = [None] * len(self.global_params)
        for k, i in enumerate(self.comp):
            full[i] = means[k]
        for k, i in enumerate(self.plain):
            full[i] = plain_means[k]
        deltas = []
        for i, p in enumerate(self.global_params):
            v = self.velocity[i]
            v.mul_(c.momentum).add_(full[i].view_as(v))
            d = (-lr) * v
            p.add_(d)
            deltas.append(d.reshape(-1).contiguous())
        pull_bytes = self._pull(deltas)
        nvals = sum(self.sizes)
        rec = {"step": self.step_no, "loss": sum(losses) / W, "lr": lr,
               "push_bytes_total": push_bytes, "pull_bytes_total": pull_bytes * W,
               "bits_per_value_push": 8.0 * push_bytes / (W * nvals),
               "bits_per_value_pull": 8.0 * pull_bytes / nvals}
        if c.eval_every and (self.step_no % c.eval_every == 0 or self.step_no == c.steps - 1):
            rec["test_acc"] = self.evaluate()
        self.log.append(rec)
        self.step_no += 1
        if record:
            return rec, grads, means, deltas
        return rec

    def _pull(self, deltas) -> int:
        """Compress each delta once (shared pull) and apply it to the replica."""
        c, dev = self.cfg, self.dev
        dc = [deltas[i] for i in self.comp]
        rep = [self.replica[i].view(-1) for i in self.comp]
        for i in self.plain:                                     # uncompressed: fp32 delta
            self.replica[i].view(-1).add_(deltas[i])
        if c.codec == "3lc":
            self.pull_ctx.compress(dc, c.s, c.use_zre)
            self.pull_ctx.decompress(rep, TLC_MODE_ACCUMULATE)
            return sum(h["payload_len"] for h in self.pull_ctx.headers())
        if c.codec == "stoch":
            total = 0
            for k, d in enumerate(dc):
                pay, hdr = self.pull_ctx.payloads[k], self.pull_ctx.hdrs[k]
                tlc_stoch_compress(d, (c.seed << 20) ^ 0xFFFFF ^ k, self.step_no, c.use_zre, pay, hdr)
                tlc_decompress(pay, hdr, d.numel(), rep[k], TLC_MODE_ACCUMULATE)
                total += parse_header(hdr)["payload_len"]
            return total
        if c.codec == "int8":
            for k, d in enumerate(dc):
                codes, hdr = tlc_int8_compress(d)
                tlc_int8_decompress(codes, hdr, d.numel(), rep[k], TLC_MODE_ACCUMULATE)
            return sum(d.numel() for d in dc)
        for k, d in enumerate(dc):
            rep[k].add_(d)
        return 4 * sum(d.numel() for d in dc)

    def run(self):
        for _ in range(self.cfg.steps - self.step_no):
            self.step()
        return self.log


def summarize(log, frac: float = 0.5) -> dict:
    """Averages over the last `frac` of the steps (the paper reports averages over training,
    Table 2) plus the final loss / accuracy."""
    tail = log[int(len(log) * (1 - frac)):]
    acc = [r["test_acc"] for r in log if "test_acc" in r]
    return {"final_loss": sum(r["loss"] for r in log[-10:]) / min(10, len(log)),
            "final_test_acc": acc[-1] if acc else None,
            "bits_per_value_push": sum(r["bits_per_value_push"] for r in tail) / len(tail),
            "bits_per_value_pull": sum(r["bits_per_value_pull"] for r in tail) / len(tail),
            "bits_per_value_push_all": sum(r["bits_per_value_push"] for r in log) / len(log),
            "bits_per_value_pull_all": sum(r["bits_per_value_pull"] for r in log) / len(log)}
