"""CIFAR ShuffleNetV2 (x1.0) client oracle -- TEST INFRASTRUCTURE ONLY (parity UNPINNED by the reference).

BASELINE.json config 4 names ShuffleNetV2 (and MobileNetV2) on CIFAR-shaped inputs; the reference has no
CNN.  This is the common CIFAR variant: 3x3 stride-1 stem to 24 channels (no max-pool),
three stages of one down-sampling block + (3, 7, 3) basic blocks with (116, 232, 464) output channels
(channel split 1/2, 1x1 - depthwise 3x3 - 1x1 branch, concatenation and a 2-group channel shuffle), a 1x1
head to 1024, 4x4 average pool and a linear classifier; fp32 on the CPU, trained with
fl_core.local_train's loop (fl_core.py:163-194) exactly like oracle/resnet.py.  rounding="bf16" rounds
where the engine stores bf16 (conv outputs, BN-ReLU outputs, block outputs) and the branch data gradients.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.nn as nn
import torch.nn.functional as F

from .flmath import batch_plan
from .mobilenet import _RoundGradBF16
from .resnet import _ID, _RoundBF16, _StraightBF16, state_keys

OUT = (116, 232, 464, 1024)
NUM = (3, 7, 3)


def shuffle(x):
    n, c, h, w = x.shape
    return x.view(n, 2, c // 2, h, w).permute(0, 2, 1, 3, 4).reshape(n, c, h, w)


class BasicBlock(nn.Module):
    def __init__(self, c):
        super().__init__()
        h = c // 2
        self.conv1 = nn.Conv2d(h, h, 1, bias=False)
        self.bn1 = nn.BatchNorm2d(h)
        self.conv2 = nn.Conv2d(h, h, 3, 1, 1, groups=h, bias=False)
        self.bn2 = nn.BatchNorm2d(h)
        self.conv3 = nn.Conv2d(h, h, 1, bias=False)
        self.bn3 = nn.BatchNorm2d(h)

    def forward(self, x, r=_ID, wq=_ID, rg=_ID):
        h = x.shape[1] // 2
        x1, x2 = x[:, :h], x[:, h:]
        b = r(F.relu(self.bn1(r(F.conv2d(rg(x2), wq(self.conv1.weight))))))
        b = r(self.bn2(r(F.conv2d(b, wq(self.conv2.weight), padding=1, groups=h))))
        b = r(F.relu(self.bn3(r(F.conv2d(b, wq(self.conv3.weight))))))
        return shuffle(torch.cat([x1, b], 1))


class DownBlock(nn.Module):
    def __init__(self, cin, cout):
        super().__init__()
        mid = cout // 2
        self.conv1 = nn.Conv2d(cin, cin, 3, 2, 1, groups=cin, bias=False)
        self.bn1 = nn.BatchNorm2d(cin)
        self.conv2 = nn.Conv2d(cin, mid, 1, bias=False)
        self.bn2 = nn.BatchNorm2d(mid)
        self.conv3 = nn.Conv2d(cin, mid, 1, bias=False)
        self.bn3 = nn.BatchNorm2d(mid)
        self.conv4 = nn.Conv2d(mid, mid, 3, 2, 1, groups=mid, bias=False)
        self.bn4 = nn.BatchNorm2d(mid)
        self.conv5 = nn.Conv2d(mid, mid, 1, bias=False)
        self.bn5 = nn.BatchNorm2d(mid)

    def forward(self, x, r=_ID, wq=_ID, rg=_ID):
        cin, mid = x.shape[1], self.conv2.weight.shape[0]
        o1 = r(self.bn1(r(F.conv2d(rg(x), wq(self.conv1.weight), stride=2, padding=1, groups=cin))))
        o1 = r(F.relu(self.bn2(r(F.conv2d(o1, wq(self.conv2.weight))))))
        o2 = r(F.relu(self.bn3(r(F.conv2d(rg(x), wq(self.conv3.weight))))))
        o2 = r(self.bn4(r(F.conv2d(o2, wq(self.conv4.weight), stride=2, padding=1, groups=mid))))
        o2 = r(F.relu(self.bn5(r(F.conv2d(o2, wq(self.conv5.weight))))))
        return shuffle(torch.cat([o1, o2], 1))


class ShuffleNetV2(nn.Module):
    def __init__(self, n_classes: int):
        super().__init__()
        self.conv1 = nn.Conv2d(3, 24, 3, 1, 1, bias=False)
        self.bn1 = nn.BatchNorm2d(24)
        cin, layers = 24, []
        for cout, n in zip(OUT[:3], NUM):
            blocks = [DownBlock(cin, cout)] + [BasicBlock(cout) for _ in range(n)]
            layers.append(nn.Sequential(*blocks))
            cin = cout
        self.layer1, self.layer2, self.layer3 = layers
        self.conv2 = nn.Conv2d(OUT[2], OUT[3], 1, bias=False)
        self.bn2 = nn.BatchNorm2d(OUT[3])
        self.linear = nn.Linear(OUT[3], n_classes)

    def forward(self, x, rounding=None):
        r = _RoundBF16.apply if rounding == "bf16" else _ID
        wq = _StraightBF16.apply if rounding == "bf16" else _ID
        rg = _RoundGradBF16.apply if rounding == "bf16" else _ID
        out = r(F.relu(self.bn1(r(F.conv2d(r(x), wq(self.conv1.weight), padding=1)))))
        for layer in (self.layer1, self.layer2, self.layer3):
            for blk in layer:
                out = blk(out, r, wq, rg)
        out = r(F.relu(self.bn2(r(F.conv2d(out, wq(self.conv2.weight))))))
        return self.linear(F.avg_pool2d(out, 4).flatten(1))


def local_train_shufflenet(params: dict[str, np.ndarray], x: np.ndarray, y: np.ndarray, num_samples: int,
                           batch_size: int, lr: float, seed, n_classes: int, max_steps: int | None = None,
                           rounding=None):
    """fl_core.local_train's loop for ShuffleNetV2 (torch CPU); returns (delta per state tensor, losses)."""
    model = ShuffleNetV2(n_classes)
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
