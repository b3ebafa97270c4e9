"""FEMNIST CNN client oracle -- TEST INFRASTRUCTURE ONLY (parity UNPINNED by the reference).

The reference ships no CNN ("parity unpinned by the
reference"; §8c: "use a torch-CPU restatement with reference batch order and
FedAvg as the builder's own oracle, labelled as such").  This module is that
restatement:

* model: LEAF FEMNIST CNN -- conv5x5 1->32 (pad 2) + ReLU + maxpool2,
  conv5x5 32->64 (pad 2) + ReLU + maxpool2, fc 3136->2048 + ReLU, fc 2048->C;
  mean softmax cross-entropy, plain SGD;
* local loop: fl_core.local_train (fl_core.py:163-194) -- the batch order is
  ``oracle.flmath.batch_plan`` (PCG64, bit-exact with the reference), one SGD
  step per batch, Δ = new − old;
* parameters in torch's canonical shapes (conv [out,in,5,5], fc [out,in],
  fc1 input flattened in torch's (c, h, w) order).

``local_train_cnn(..., rounding=None)`` is plain fp32 (torch CPU).  With
``rounding=bf16`` it rounds at exactly the points the B200 engine stores
bf16 (inputs, weight shadows, activations, gradients between layers), which
makes a single step comparable at bf16-ulp level; the manual backward is
pinned to torch autograd by ``tests/test_cnn_oracle.py``.
"""

from __future__ import annotations

import math

import numpy as np
import torch
import torch.nn.functional as F

from .flmath import batch_plan

HID = 2048


def init_params(n_classes: int, seed: int) -> dict[str, np.ndarray]:
    """Uniform(-1/sqrt(fan_in), +) init (torch's default bound), float64, numpy PCG64."""
    rng = np.random.default_rng(seed)
    shapes = [("conv1.weight", (32, 1, 5, 5), 25), ("conv1.bias", (32,), 25),
              ("conv2.weight", (64, 32, 5, 5), 800), ("conv2.bias", (64,), 800),
              ("fc1.weight", (HID, 3136), 3136), ("fc1.bias", (HID,), 3136),
              ("fc2.weight", (n_classes, HID), HID), ("fc2.bias", (n_classes,), HID)]
    out = {}
    for name, shape, fan_in in shapes:
        b = 1.0 / math.sqrt(fan_in)
        out[name] = rng.uniform(-b, b, size=shape)
    return out


def _bf16(t: torch.Tensor) -> torch.Tensor:
    return t.to(torch.bfloat16).to(torch.float32)


def _id(t: torch.Tensor) -> torch.Tensor:
    return t


def _pool_fwd(a: torch.Tensor):
    """2x2 max pool [N,C,H,W]; window index of the first max in row-major order."""
    n, c, h, w = a.shape
    win = a.reshape(n, c, h // 2, 2, w // 2, 2).permute(0, 1, 2, 4, 3, 5).reshape(n, c, h // 2, w // 2, 4)
    m = win.max(dim=-1).values
    first = (win == m.unsqueeze(-1)).float().argmax(dim=-1)  # first max
    return m, first


def _pool_bwd(g: torch.Tensor, first: torch.Tensor, a: torch.Tensor) -> torch.Tensor:
    """Route g to the first-max position, ReLU mask (a > 0) -> [N,C,H,W]."""
    n, c, ho, wo = g.shape
    onehot = F.one_hot(first, 4).to(g.dtype)  # [n,c,ho,wo,4]
    win = (g.unsqueeze(-1) * onehot).reshape(n, c, ho, wo, 2, 2).permute(0, 1, 2, 4, 3, 5)
    out = win.reshape(n, c, 2 * ho, 2 * wo)
    return out * (a > 0)


def step(p: dict[str, torch.Tensor], x: torch.Tensor, y: torch.Tensor, lr: float, n_classes: int,
         q=_id) -> float:
    """One SGD step on batch (x [b,784], y [b]) in place; returns the mean CE loss."""
    b = x.shape[0]
    xi = q(x.reshape(b, 1, 28, 28))
    w1, w2 = q(p["conv1.weight"]), q(p["conv2.weight"])
    f1, f2 = q(p["fc1.weight"]), q(p["fc2.weight"])
    # forward (im2col formulation; fp32 accumulation)
    cols1 = F.unfold(xi, 5, padding=2)                                   # [b, 25, 784]
    z1 = torch.einsum("bkp,ok->bop", cols1, w1.reshape(32, 25)) + p["conv1.bias"][None, :, None]
    a1 = q(torch.relu(z1).reshape(b, 32, 28, 28))
    p1, first1 = _pool_fwd(a1)
    cols2 = F.unfold(p1, 5, padding=2)                                   # [b, 800, 196]
    z2 = torch.einsum("bkp,ok->bop", cols2, w2.reshape(64, 800)) + p["conv2.bias"][None, :, None]
    a2 = q(torch.relu(z2).reshape(b, 64, 14, 14))
    p2, first2 = _pool_fwd(a2)
    flat = p2.reshape(b, 3136)
    h = q(torch.relu(flat @ f1.T + p["fc1.bias"]))
    logits = h @ f2.T + p["fc2.bias"]
    lse = torch.logsumexp(logits, dim=1)
    loss = float((lse - logits[torch.arange(b), y]).mean())
    prob = torch.softmax(logits, dim=1)
    dl = q((prob - F.one_hot(y, n_classes).float()) / b)
    # backward (each gradient uses the step's pre-update weights)
    g_fc2 = dl.T @ h
    g_b2 = dl.sum(0)
    dh = q((dl @ f2) * (h > 0))
    g_fc1 = dh.T @ flat
    g_b1 = dh.sum(0)
    dp2 = q(dh @ f1).reshape(b, 64, 7, 7)
    da2 = _pool_bwd(dp2, first2, a2)                                      # exact copy of bf16 values
    da2m = da2.reshape(b, 64, 196)
    g_c2 = torch.einsum("bop,bkp->ok", da2m, cols2).reshape(64, 32, 5, 5)
    g_bc2 = da2m.sum((0, 2))
    dcols2 = q(torch.einsum("bop,ok->bkp", da2m, w2.reshape(64, 800)))   # [b, 800, 196]
    dp1 = F.fold(dcols2, (14, 14), 5, padding=2)                         # fp32 sum over taps
    da1 = q(_pool_bwd(dp1, first1, a1))
    da1m = da1.reshape(b, 32, 784)
    g_c1 = torch.einsum("bop,bkp->ok", da1m, cols1).reshape(32, 1, 5, 5)
    g_bc1 = da1m.sum((0, 2))
    for name, g in (("conv1.weight", g_c1), ("conv1.bias", g_bc1), ("conv2.weight", g_c2), ("conv2.bias", g_bc2),
                    ("fc1.weight", g_fc1), ("fc1.bias", g_b1), ("fc2.weight", g_fc2), ("fc2.bias", g_b2)):
        p[name] -= lr * g
    return loss


def local_train_cnn(params: dict[str, np.ndarray], x: np.ndarray, y: np.ndarray, num_samples: int,
                    batch_size: int, lr: float, seed, n_classes: int, rounding=None,
                    max_steps: int | None = None) -> tuple[dict[str, np.ndarray], list[float]]:
    """fl_core.local_train's loop (fl_core.py:163-194) for the CNN; returns (Δ per tensor, losses).

    Δ = (new − old) in fp32 master precision, like the engine's deltas.
    """
    q = _bf16 if rounding == "bf16" else _id
    p = {k: torch.tensor(v, dtype=torch.float32) for k, v in params.items()}
    start = {k: v.clone() for k, v in p.items()}
    losses = []
    if len(y):
        xt = torch.tensor(np.asarray(x, dtype=np.float32))
        yt = torch.tensor(np.asarray(y, dtype=np.int64))
        plan = batch_plan(len(y), num_samples, batch_size, seed)
        for s, idx in enumerate(plan):
            if max_steps is not None and s >= max_steps:
                break
            ix = torch.tensor(idx, dtype=torch.int64)
            losses.append(step(p, xt[ix], yt[ix], lr, n_classes, q))
    return {k: (p[k] - start[k]).numpy() for k in p}, losses


def forward_logits(params: dict[str, np.ndarray], x: np.ndarray) -> np.ndarray:
    """fp32 forward of the canonical model (for accuracy checks)."""
    p = {k: torch.tensor(v, dtype=torch.float32) for k, v in params.items()}
    xt = torch.tensor(np.asarray(x, dtype=np.float32)).reshape(-1, 1, 28, 28)
    a = F.max_pool2d(torch.relu(F.conv2d(xt, p["conv1.weight"], p["conv1.bias"], padding=2)), 2)
    a = F.max_pool2d(torch.relu(F.conv2d(a, p["conv2.weight"], p["conv2.bias"], padding=2)), 2)
    h = torch.relu(a.reshape(a.shape[0], -1) @ p["fc1.weight"].T + p["fc1.bias"])
    return (h @ p["fc2.weight"].T + p["fc2.bias"]).numpy()
