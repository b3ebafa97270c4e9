"""CIFAR ResNet-18 client oracle -- TEST INFRASTRUCTURE ONLY (parity UNPINNED by the reference).

The reference ships no CNN ("parity unpinned by the reference"; §8c: "use a torch-CPU
restatement with reference batch order and FedAvg as the builder's own oracle").  BASELINE.json config 3
names ResNet-18 on CIFAR-shaped 32x32x3 inputs; this is the usual CIFAR variant (3x3 stem, no max-pool,
BasicBlocks 64-128-256-512 with 1x1 projection shortcuts, batch norm in training mode, global average
pool, linear classifier), fp32 on the CPU, trained with fl_core.local_train's loop (fl_core.py:163-194):
the PCG64 batch order of ``oracle.flmath.batch_plan``, plain SGD, Δ = new − old over the whole state
(weights and BN running statistics, which FedAvg averages like torch's state_dict).
Input rows are NHWC fp32 [32][32][3] flattened (3072 features), as the engine stores them.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.nn as nn
import torch.nn.functional as F

from .flmath import batch_plan

BLOCKS = [(64, 64, 1), (64, 64, 1), (64, 128, 2), (128, 128, 1), (128, 256, 2), (256, 256, 1), (256, 512, 2),
          (512, 512, 1)]


class _RoundBF16(torch.autograd.Function):
    """Round to bf16 in the forward and round the incoming gradient in the backward -- the engine stores
    this activation and its gradient in bf16 (csrc/resnet.cu)."""

    @staticmethod
    def forward(ctx, x):
        return x.to(torch.bfloat16).float()

    @staticmethod
    def backward(ctx, g):
        return g.to(torch.bfloat16).float()


class _StraightBF16(torch.autograd.Function):
    """bf16 weight shadow: round in the forward, pass the gradient to the fp32 master unchanged."""

    @staticmethod
    def forward(ctx, w):
        return w.to(torch.bfloat16).float()

    @staticmethod
    def backward(ctx, g):
        return g


_ID = (lambda t: t)


class BasicBlock(nn.Module):
    def __init__(self, cin, cout, s):
        super().__init__()
        self.conv1 = nn.Conv2d(cin, cout, 3, s, 1, bias=False)
        self.bn1 = nn.BatchNorm2d(cout)
        self.conv2 = nn.Conv2d(cout, cout, 3, 1, 1, bias=False)
        self.bn2 = nn.BatchNorm2d(cout)
        self.shortcut = nn.Sequential()
        if s != 1 or cin != cout:
            self.shortcut = nn.Sequential(nn.Conv2d(cin, cout, 1, s, bias=False), nn.BatchNorm2d(cout))

    def forward(self, x, r=_ID, wq=_ID):
        c1 = r(F.conv2d(x, wq(self.conv1.weight), stride=self.conv1.stride, padding=1))
        a1 = r(F.relu(self.bn1(c1)))
        c2 = r(F.conv2d(a1, wq(self.conv2.weight), padding=1))
        if len(self.shortcut):
            conv, bn = self.shortcut[0], self.shortcut[1]
            sc = bn(r(F.conv2d(x, wq(conv.weight), stride=conv.stride)))
        else:
            sc = x
        return r(F.relu(self.bn2(c2) + sc))


class ResNet18(nn.Module):
    def __init__(self, n_classes: int):
        super().__init__()
        self.conv1 = nn.Conv2d(3, 64, 3, 1, 1, bias=False)
        self.bn1 = nn.BatchNorm2d(64)
        layers = [BasicBlock(ci, co, s) for ci, co, s in BLOCKS]
        self.layer1, self.layer2 = nn.Sequential(*layers[0:2]), nn.Sequential(*layers[2:4])
        self.layer3, self.layer4 = nn.Sequential(*layers[4:6]), nn.Sequential(*layers[6:8])
        self.linear = nn.Linear(512, n_classes)

    def forward(self, x, rounding=None):
        r = _RoundBF16.apply if rounding == "bf16" else _ID
        wq = _StraightBF16.apply if rounding == "bf16" else _ID
        out = r(F.relu(self.bn1(r(F.conv2d(r(x), wq(self.conv1.weight), padding=1)))))
        for layer in (self.layer1, self.layer2, self.layer3, self.layer4):
            for blk in layer:
                out = blk(out, r, wq)
        return self.linear(F.avg_pool2d(out, 4).flatten(1))


def state_keys(model: nn.Module) -> list[str]:
    return [k for k in model.state_dict() if not k.endswith("num_batches_tracked")]


def local_train_resnet(params: dict[str, np.ndarray], x: np.ndarray, y: np.ndarray, num_samples: int,
                       batch_size: int, lr: float, seed, n_classes: int, max_steps: int | None = None,
                       rounding=None):
    """fl_core.local_train's loop for ResNet-18 (torch CPU); returns (Δ per state tensor, losses).

    rounding=None: plain fp32.  rounding="bf16": bf16 weights (straight-through to the fp32 master) and
    bf16 activations / layer-boundary gradients exactly where the engine stores them (input, conv
    outputs, post-ReLU activations, block outputs); batch norm in fp32 on the rounded inputs."""
    model = ResNet18(n_classes)
    sd = model.state_dict()
    for k in state_keys(model):
        sd[k].copy_(torch.tensor(params[k], dtype=torch.float32))
    model.train()
    opt = torch.optim.SGD(model.parameters(), lr=lr)
    start = {k: v.clone() for k, v in model.state_dict().items()}
    losses = []
    if len(y):
        xt = torch.tensor(np.asarray(x, dtype=np.float32)).reshape(-1, 32, 32, 3).permute(0, 3, 1, 2).contiguous()
        yt = torch.tensor(np.asarray(y, dtype=np.int64))
        for s, idx in enumerate(batch_plan(len(y), num_samples, batch_size, seed)):
            if max_steps is not None and s >= max_steps:
                break
            ix = torch.tensor(idx, dtype=torch.int64)
            opt.zero_grad(set_to_none=True)
            loss = F.cross_entropy(model(xt[ix], rounding), yt[ix])
            loss.backward()
            opt.step()
            losses.append(float(loss.detach()))
    end = model.state_dict()
    return {k: (end[k] - start[k]).numpy().astype(np.float64) for k in state_keys(model)}, losses
