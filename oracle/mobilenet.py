"""CIFAR MobileNetV2 client oracle -- TEST INFRASTRUCTURE ONLY (parity UNPINNED by the reference).

The reference ships no CNN ("parity unpinned by the reference"; §8c: torch-CPU restatement
with the reference batch order and FedAvg as the builder's own oracle).  BASELINE.json config 4 names
MobileNetV2 on CIFAR-shaped 32x32x3 inputs; this is the common CIFAR variant (3x3 stride-1 stem with 32
channels, 17 inverted-residual blocks from the (t, c, n, s) table with stride 1 in the second stage, ReLU,
identity / 1x1-conv-BN shortcut at stride 1, 1x1 head to 1280, 4x4 average pool, linear), fp32 on the CPU,
trained with fl_core.local_train's loop (fl_core.py:163-194) exactly like oracle/resnet.py.
Input rows are NHWC fp32 [32][32][3] flattened (3072 features), as the engine stores them.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.nn as nn
import torch.nn.functional as F

from .flmath import batch_plan
from .resnet import _ID, _RoundBF16, _StraightBF16, state_keys


class _RoundGradBF16(torch.autograd.Function):
    """Identity in the forward; rounds the gradient to bf16 in the backward -- the engine stores each
    convolution's data gradient in bf16 before it is summed with the other branch (csrc/resnet.cu, mb)."""

    @staticmethod
    def forward(ctx, x):
        return x

    @staticmethod
    def backward(ctx, g):
        return g.to(torch.bfloat16).float()

CFG = [(1, 16, 1, 1), (6, 24, 2, 1), (6, 32, 3, 2), (6, 64, 4, 2), (6, 96, 3, 1), (6, 160, 3, 2), (6, 320, 1, 1)]


class Block(nn.Module):
    def __init__(self, cin, cout, expansion, stride):
        super().__init__()
        self.stride = stride
        planes = expansion * cin
        self.conv1 = nn.Conv2d(cin, planes, 1, bias=False)
        self.bn1 = nn.BatchNorm2d(planes)
        self.conv2 = nn.Conv2d(planes, planes, 3, stride, 1, groups=planes, bias=False)
        self.bn2 = nn.BatchNorm2d(planes)
        self.conv3 = nn.Conv2d(planes, cout, 1, bias=False)
        self.bn3 = nn.BatchNorm2d(cout)
        self.shortcut = nn.Sequential()
        if stride == 1 and cin != cout:
            self.shortcut = nn.Sequential(nn.Conv2d(cin, cout, 1, bias=False), nn.BatchNorm2d(cout))

    def forward(self, x, r=_ID, wq=_ID, rg=_ID):
        e = r(F.conv2d(rg(x), wq(self.conv1.weight)))
        ea = r(F.relu(self.bn1(e)))
        d = r(F.conv2d(ea, wq(self.conv2.weight), stride=self.stride, padding=1, groups=ea.shape[1]))
        da = r(F.relu(self.bn2(d)))
        out = self.bn3(r(F.conv2d(da, wq(self.conv3.weight))))
        if self.stride == 1:
            if len(self.shortcut):
                conv, bn = self.shortcut[0], self.shortcut[1]
                out = out + bn(r(F.conv2d(rg(x), wq(conv.weight))))
            else:
                out = out + x
        return r(out)


class MobileNetV2(nn.Module):
    def __init__(self, n_classes: int):
        super().__init__()
        self.conv1 = nn.Conv2d(3, 32, 3, 1, 1, bias=False)
        self.bn1 = nn.BatchNorm2d(32)
        layers, cin = [], 32
        for t, c, n, s in CFG:
            for i in range(n):
                layers.append(Block(cin, c, t, s if i == 0 else 1))
                cin = c
        self.layers = nn.Sequential(*layers)
        self.conv2 = nn.Conv2d(320, 1280, 1, bias=False)
        self.bn2 = nn.BatchNorm2d(1280)
        self.linear = nn.Linear(1280, n_classes)

    def forward(self, x, rounding=None):
        r = _RoundBF16.apply if rounding == "bf16" else _ID
        wq = _StraightBF16.apply if rounding == "bf16" else _ID
        rg = _RoundGradBF16.apply if rounding == "bf16" else _ID
        out = r(F.relu(self.bn1(r(F.conv2d(r(x), wq(self.conv1.weight), padding=1)))))
        for blk in self.layers:
            out = blk(out, r, wq, rg if (blk.stride == 1) else _ID)
        out = r(F.relu(self.bn2(r(F.conv2d(out, wq(self.conv2.weight))))))
        return self.linear(F.avg_pool2d(out, 4).flatten(1))


def local_train_mobilenet(params: dict[str, np.ndarray], x: np.ndarray, y: np.ndarray, num_samples: int,
                          batch_size: int, lr: float, seed, n_classes: int, max_steps: int | None = None,
                          rounding=None):
    """fl_core.local_train's loop for MobileNetV2 (torch CPU); returns (Δ per state tensor, losses).
    rounding as oracle.resnet.local_train_resnet."""
    model = MobileNetV2(n_classes)
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
