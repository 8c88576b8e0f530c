"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic (no max, no quantization, no
encoding): it only draws fp32 state-change tensors with the shapes and value
distributions of the paper's workloads ("input recipe").

* The paper's state changes are per-layer fp32 gradients / model deltas "centered
  around zero" of ResNet-110 on CIFAR-10; BN tensors are
  not compressed, so workloads keep the ndim >= 2 tensors (R19).
* Every draw is numpy PCG64 keyed by a tuple (SeedSequence), so each
  (config, layer, rank, step) stream is independent and reproducible.
"""
from __future__ import annotations

import numpy as np

# --------------------------------------------------------------------------- tensor lists
# ResNet-110 for CIFAR (He et al. 2016, option-A shortcuts): 3 stages x 18 basic
# blocks, widths 16/32/64; conv1 3->16, fc 64->10.  ndim >= 2 tensors only.
RESNET110_SIZES = (
    [3 * 16 * 9]
    + [16 * 16 * 9] * 36
    + [32 * 16 * 9] + [32 * 32 * 9] * 35
    + [64 * 32 * 9] + [64 * 64 * 9] * 35
    + [10 * 64]
)


def _resnet50_sizes():
    out = [64 * 3 * 7 * 7]
    inp = 64
    for width, blocks in ((64, 3), (128, 4), (256, 6), (512, 3)):
        for b in range(blocks):
            out += [width * inp, width * width * 9, 4 * width * width]
            if b == 0:
                out.append(4 * width * inp)          # downsample 1x1
            inp = 4 * width
    out.append(1000 * 2048)
    return out


RESNET50_SIZES = _resnet50_sizes()

# BERT-large (HF BertForPreTraining, 24 x 1024, FFN 4096), ndim >= 2, decoder tied.
BERT_LARGE_SIZES = (
    [30522 * 1024, 512 * 1024, 2 * 1024]
    + [1024 * 1024, 1024 * 1024, 1024 * 1024, 1024 * 1024, 4096 * 1024, 1024 * 4096] * 24
    + [1024 * 1024, 1024 * 1024, 2 * 1024]
)

assert len(RESNET110_SIZES) == 110 and sum(RESNET110_SIZES) == 1_719_856
assert len(RESNET50_SIZES) == 54 and sum(RESNET50_SIZES) == 25_502_912
assert len(BERT_LARGE_SIZES) == 150 and sum(BERT_LARGE_SIZES) == 335_869_952

MODELS = {"resnet110": RESNET110_SIZES, "resnet50": RESNET50_SIZES, "bert-large": BERT_LARGE_SIZES}


# --------------------------------------------------------------------------- generators
def rng(*key: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([int(k) for k in key])))


def gaussian(n: int, *key: int) -> np.ndarray:
    """N(0,1) fp32, the 'gauss' family (C1, C3 gauss-steady)."""
    return rng(*key).standard_normal(n, dtype=np.float32)


def layer_gradient(n: int, mu: float, *key: int) -> np.ndarray:
    """One layer's state change: g = mu_l + z, z ~ N(0,1) fresh per step (C2/C4/C5)."""
    g = rng(*key).standard_normal(n, dtype=np.float32)
    g += np.float32(mu)
    return g


def layer_means(sizes, *key: int) -> np.ndarray:
    """Per-layer offsets mu_l = 0.3 * N(0,1), fixed for a run."""
    return (0.3 * rng(*key).standard_normal(len(sizes))).astype(np.float32)


def model_step(model: str, step: int, rank: int = 0, cfg: int = 2):
    """All tensors of ``model`` for one (rank, step): list of fp32 arrays."""
    sizes = MODELS[model]
    mus = layer_means(sizes, cfg, 10_000 + len(sizes))
    return [layer_gradient(n, mus[l], cfg, rank, l, step) for l, n in enumerate(sizes)]


def model_step_torch(model: str, step: int, rank: int, device, cfg: int = 5):
    """Device-side draw of one (rank, step) state change for every tensor of
    ``model``: g = mu_l + z with torch's seeded Philox generator on ``device``
    (bench-only, for the 336M-value BERT-large lists; same distribution as
    model_step, different stream)."""
    import torch

    sizes = MODELS[model]
    mus = layer_means(sizes, cfg, 10_000 + len(sizes))
    g = torch.Generator(device=device)
    g.manual_seed(int(np.random.SeedSequence([cfg, rank, step]).generate_state(1)[0]))
    out = []
    for l, n in enumerate(sizes):
        x = torch.randn(n, generator=g, device=device, dtype=torch.float32)
        x += float(mus[l])
        out.append(x)
    return out


def zeros(n: int) -> np.ndarray:
    """'zeros' family: every state change is 0 (P:546-548's all-zero tensor)."""
    return np.zeros(n, dtype=np.float32)


def dense(n: int, s: float, A: float = 1.0, *key: int) -> np.ndarray:
    """'dense' family: |t| in [A*(s/2 + 2^-20), A] with random sign and one element
    exactly +A, so every |t| / (A*s) > 1/2 (no zero value after quantization)."""
    g = rng(*(key or (3, 1)))
    lo = np.float32(A) * (np.float32(s) / np.float32(2) + np.float32(2.0 ** -20))
    mag = g.uniform(float(lo), float(A), size=n).astype(np.float32)
    sign = np.where(g.integers(0, 2, size=n) == 0, np.float32(-1), np.float32(1))
    t = (mag * sign).astype(np.float32)
    t[g.integers(0, n)] = np.float32(A)
    return t


def runs_adversarial(n: int, A: float = 1.0, *key: int) -> np.ndarray:
    """'runs' family.  The compressor groups elements {j, j+P, ..., j+4P},
    P = ceil(n/5).  Pick, per group j, either an all-zero group or a
    'separator' group whose first element is +-A, laying runs of all-zero groups
    with lengths 1..100 and 14k-1, 14k, 14k+1, so run boundaries fall at every
    offset mod 14 and across any tile edge."""
    g = rng(*(key or (3, 2)))
    P = -(-n // 5)
    t = np.zeros(n, dtype=np.float32)
    j = 0
    menu = list(range(1, 101)) + [14 * k + d for k in range(1, 40) for d in (-1, 0, 1)]
    while j < P:
        run = int(menu[g.integers(0, len(menu))])
        j += run                                  # all-zero groups
        if j >= P:
            break
        seps = int(g.integers(1, 4))
        for _ in range(seps):
            if j >= P:
                break
            t[j] = np.float32(A) if g.integers(0, 2) else np.float32(-A)
            j += 1
    if not np.any(t):
        t[0] = np.float32(A)
    return t


def family(name: str, n: int, s: float, seed: int = 3) -> np.ndarray:
    if name == "gauss":
        return gaussian(n, seed, 0)
    if name == "zeros":
        return zeros(n)
    if name == "dense":
        return dense(n, s, 1.0, seed, 1)
    if name == "runs":
        return runs_adversarial(n, 1.0, seed, 2)
    raise ValueError(name)


def family_torch(name: str, n: int, s: float, device, seed: int = 3, step: int = 0):
    """Device-side draw of a C3 family (bench-only, for the 2^20..2^30 sweep): the same
    distributions as ``family`` -- gauss N(0,1); zeros; dense |t| in [s/2 + 2^-20, 1]
    with random sign and one element exactly +1; runs: all-zero quartic groups in runs
    of 1..100 and 14k-1/14k/14k+1 between 1-3 separator groups whose partition-0
    element is +-1 -- from torch's seeded Philox generator (other streams than the
    numpy generators; no parity use)."""
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(int(np.random.SeedSequence([seed, n, step, len(name)]).generate_state(1)[0]))
    if name == "gauss":
        return torch.randn(n, generator=g, device=device, dtype=torch.float32)
    if name == "zeros":
        return torch.zeros(n, device=device, dtype=torch.float32)
    if name == "dense":
        lo = float(np.float32(s) / np.float32(2) + np.float32(2.0 ** -20))
        t = torch.rand(n, generator=g, device=device, dtype=torch.float32) * (1.0 - lo) + lo
        t = t.clamp_(min=lo, max=1.0)
        t *= torch.randint(0, 2, (n,), generator=g, device=device, dtype=torch.int8).float() * 2 - 1
        t[n // 2] = 1.0
        return t
    if name == "runs":
        P = -(-n // 5)
        menu = torch.tensor(list(range(1, 101)) + [14 * k + d for k in range(1, 40) for d in (-1, 0, 1)],
                            device=device)
        # blocks of (run of zero groups, 1-3 separators); enough blocks to cover P
        K = P // 40 + 16
        run = menu[torch.randint(0, menu.numel(), (K,), generator=g, device=device)]
        sep = torch.randint(1, 4, (K,), generator=g, device=device)
        start = torch.cumsum(run + sep, 0) - sep                     # first separator of each block
        groups = torch.zeros(P + 4, device=device, dtype=torch.float32)
        for k in range(3):
            idx = start + k
            ok = (k < sep) & (idx < P)
            sign = torch.randint(0, 2, (K,), generator=g, device=device).float() * 2 - 1
            groups[idx[ok]] = sign[ok]
        t = torch.zeros(n, device=device, dtype=torch.float32)
        t[:P] = groups[:P]                                           # partition 0 of each group
        if not bool(t.any()):
            t[0] = 1.0
        return t
    raise ValueError(name)


def blobs(n_train: int, n_test: int, dim: int, classes: int, std: float, *key: int):
    """Desk-scale classification task of the training simulator (the
    stand-in for CIFAR-10): class c is centred at a seeded random unit-norm vector
    scaled by 2.0, points are centre + std * N(0, 1).  Returns fp32 (x_train,
    y_train, x_test, y_test); labels are stratified (n/classes per class)."""
    g = rng(*(key or (9, 0)))
    centers = g.standard_normal((classes, dim))
    centers = (2.0 * centers / np.linalg.norm(centers, axis=1, keepdims=True)).astype(np.float32)

    def draw(n):
        y = np.arange(n) % classes
        g.shuffle(y)
        x = centers[y] + np.float32(std) * g.standard_normal((n, dim)).astype(np.float32)
        return x.astype(np.float32), y.astype(np.int64)

    xtr, ytr = draw(n_train)
    xte, yte = draw(n_test)
    return xtr, ytr, xte, yte
