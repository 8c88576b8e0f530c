"""W-virtual-rank parameter-server exchange oracle (X1-X6) -- TEST INFRASTRUCTURE.

Follows the paper's push/pull step (fig. push-and-pull) with the
per-context compression of Sec. 3, in one process, over plain numpy arrays and
the C oracle's compress/decompress (oracle/tlc_oracle.c):

X1  plan: contexts (tensor, lo, hi, owner) -- reading R17, written here
    independently of the product's C++ plan.
X2  every rank r compresses every context c with push_err[r][c] (Fig. steps 1-4).
X3  the owner sums the W decompressed pushes in rank order starting from +0,
    adding M_w*q_w only where q_w != 0 (R15, R16), then divides by W in fp32
    ("average the gradients").  A context with a failed push (status
    not OK: NaN/Inf in a rank's u, or M overflow) has a NaN mean (reading R24).
X4  delta = mean (identity update in benchmarks, R18).
X5  the owner compresses delta[c] ONCE with pull_err[c] (shared pull).
X6  every rank applies every owner's payload to its full-size output with
    decompress-ACCUMULATE; all ranks end bit-identical.  A context whose shared
    pull failed (R24: its NaN mean raises NONFINITE) is left untouched.
"""
from __future__ import annotations

import numpy as np

from . import compress, decompress

f32 = np.float32


def plan(sizes, W):
    """R17: tensors larger than cap = ceil(N/W) are cut into ceil(n/cap) shards whose
    lengths differ by at most one (the first n mod m shards one longer); contexts are
    assigned largest first (stable in context order) to the least-loaded rank, the
    lowest rank winning ties."""
    N = sum(int(n) for n in sizes)
    cap = max(1, -(-N // W))
    ctx = []
    for t, n in enumerate(sizes):
        n = int(n)
        if n == 0:
            continue
        m = -(-n // cap) if n > cap else 1
        base, rem = divmod(n, m)
        lo = 0
        for k in range(m):
            ln = base + (1 if k < rem else 0)
            ctx.append([t, lo, lo + ln, -1])
            lo += ln
    order = sorted(range(len(ctx)), key=lambda k: -(ctx[k][2] - ctx[k][1]))   # stable
    load = [0] * W
    for k in order:
        r = min(range(W), key=lambda q: (load[q], q))
        ctx[k][3] = r
        load[r] += ctx[k][2] - ctx[k][1]
    return [tuple(c) for c in ctx]


class VirtualPS:
    """State of a W-rank exchange: push error buffers per (rank, context), pull error
    buffers per context (held by its owner)."""

    def __init__(self, sizes, W, ctx=None):
        """ctx: an explicit list of (tensor, lo, hi, owner) contexts instead of plan(sizes, W)
        (tests replay a few contexts of a large plan on their own: contexts are independent)."""
        self.sizes, self.W = [int(n) for n in sizes], W
        self.ctx = [tuple(c) for c in ctx] if ctx is not None else plan(self.sizes, W)
        self.push_err = [[np.zeros(hi - lo, f32) for (_, lo, hi, _) in self.ctx] for _ in range(W)]
        self.pull_err = [np.zeros(hi - lo, f32) for (_, lo, hi, _) in self.ctx]

    def push(self, grads, s, use_zre=True):
        """X2-X4.  grads[r][t]: rank r's state change of tensor t.  Returns
        (means per context, push payloads[r][c])."""
        W = self.W
        sent = [[compress(grads[r][t][lo:hi], self.push_err[r][c], s, use_zre)
                 for c, (t, lo, hi, _) in enumerate(self.ctx)] for r in range(W)]
        means = []
        for c, (t, lo, hi, owner) in enumerate(self.ctx):
            if any(sent[w][c].status != 0 for w in range(W)):    # R24
                means.append(np.full(hi - lo, np.nan, f32))
                continue
            acc = np.zeros(hi - lo, f32)                     # +0
            for w in range(W):                                # rank order
                p = sent[w][c]
                st, acc = decompress(p.payload, use_zre, p.M, hi - lo, out=acc, accumulate=True)
                assert st == 0
            means.append((acc / f32(W)).astype(f32))          # IEEE fp32 division
        return means, sent

    def pull(self, deltas, outs, s, use_zre=True):
        """X5-X6.  deltas[c]: the owner's model delta of context c; outs[r][t]:
        rank r's full-size outputs, updated in place."""
        shared = [compress(deltas[c], self.pull_err[c], s, use_zre) for c in range(len(self.ctx))]
        for r in range(self.W):
            for c, (t, lo, hi, owner) in enumerate(self.ctx):
                p = shared[c]
                if p.status != 0:                             # R24: nothing to apply
                    continue
                view = outs[r][t][lo:hi].copy()
                st, view = decompress(p.payload, use_zre, p.M, hi - lo, out=view, accumulate=True)
                assert st == 0
                outs[r][t][lo:hi] = view
        return shared

    def step(self, grads, outs, s, use_zre=True):
        means, sent = self.push(grads, s, use_zre)
        shared = self.pull(means, outs, s, use_zre)
        return means, sent, shared
