"""On-device synthetic federated data at fleet scale.

The reference generates the whole dataset on the host in fp64 from one PCG64
stream (fl_core.py:41-59) and partitions it with per-client Dirichlet class
mixes drawn without replacement (fl_core.py:62-115).  At config-3/4 scale
(1000+ clients) that is minutes of host work and tens of GB of fp64.

Here the same *distributions* are produced directly in HBM:
  * class means ~ N(0, 1) * 3, features = mean[label] + N(0, 1)  (fl_core.py:47-55)
  * per-client class counts = floor(Dir(alpha) * n_i) with the integer
    remainder given to the largest fractional parts, stable order
    (fl_core.py:89-95) -- drawn on the host (O(clients x classes), cheap)
  * the dataset is generated with exactly sum_i counts[i][c] rows of class c,
    so every client's quota is met without the reference's "richest pool"
    shortfall path (fl_core.py:103-108), and rows are assigned to clients by a
    per-class random permutation on the device, then packed contiguously
    (client shards back to back) for the TMA row gather.
Values are NOT bit-identical to the reference (a sequential host PCG64 stream
cannot be reproduced in parallel); parity tests use the host generator at
small sizes (SURVEY §7 hard parts, item 5).
"""

from __future__ import annotations

import numpy as np
import torch

from .training import device


def dirichlet_counts(sample_counts: list[int], n_classes: int, alpha: float, seed: int) -> np.ndarray:
    """[clients, classes] int64 quotas: floor(Dir(alpha) * n) + largest-remainder (fl_core.py:89-95)."""
    if alpha <= 0:
        raise ValueError("alpha must be > 0")
    rng = np.random.default_rng(seed)
    out = np.zeros((len(sample_counts), n_classes), dtype=np.int64)
    for i, n in enumerate(sample_counts):
        mix = rng.dirichlet([alpha] * n_classes)
        q = np.floor(mix * n).astype(np.int64)
        extra = int(n - q.sum())
        for c in np.argsort(-(mix * n - q), kind="stable")[:extra]:
            q[c] += 1
        out[i] = q
    return out


class DeviceFleetData:
    """Client shards (packed, fp32) + test set generated in HBM.

    Attributes mirror DeviceFederation.from_arrays' inputs: x, y, offsets
    (client id -> (row offset, n_rows)), x_test, y_test.
    """

    def __init__(self, client_ids: list[str], sample_counts: list[int], n_features: int, n_classes: int,
                 alpha: float, seed: int, n_test: int, chunk_rows: int = 1 << 20):
        dev = device()
        self.n_features, self.n_classes = n_features, n_classes
        counts = dirichlet_counts(sample_counts, n_classes, alpha, seed)
        per_class = counts.sum(axis=0)                                     # rows needed per class
        g = torch.Generator(device=dev).manual_seed(int(seed) & 0x7FFFFFFFFFFFFFFF)
        self.means = torch.randn(n_classes, n_features, device=dev, generator=g) * 3.0
        n_total = int(per_class.sum())
        # labels grouped by class, then each class block shuffled independently
        y_sorted = torch.repeat_interleave(torch.arange(n_classes, device=dev),
                                           torch.from_numpy(per_class).to(dev))
        class_start = np.concatenate([[0], np.cumsum(per_class)[:-1]])
        # client i takes rows [class_start[c] + cum_i(c), + counts[i][c]) of each class block, after a
        # per-class permutation; packing order = client order, classes ascending inside a client
        perm = torch.empty(n_total, dtype=torch.int64, device=dev)
        for c in range(n_classes):
            a, n = int(class_start[c]), int(per_class[c])
            if n:
                perm[a:a + n] = a + torch.randperm(n, device=dev, generator=g)
        take = np.cumsum(counts, axis=0) - counts                          # per-client offset within class
        src = []
        for i in range(len(sample_counts)):
            for c in range(n_classes):
                k = int(counts[i][c])
                if k:
                    a = int(class_start[c] + take[i][c])
                    src.append(perm[a:a + k])
        order = torch.cat(src) if src else torch.zeros(0, dtype=torch.int64, device=dev)
        self.y = y_sorted[order].to(torch.int32).contiguous()
        self.x = torch.empty(n_total, n_features, device=dev)
        for s in range(0, n_total, chunk_rows):
            e = min(s + chunk_rows, n_total)
            self.x[s:e] = self.means[self.y[s:e].long()] + torch.randn(e - s, n_features, device=dev, generator=g)
        self.offsets, at = {}, 0
        for cid, n in zip(client_ids, sample_counts):
            self.offsets[cid] = (at, int(n))
            at += int(n)
        yt = torch.randint(0, n_classes, (n_test,), device=dev, generator=g, dtype=torch.int32)
        self.x_test = self.means[yt.long()] + torch.randn(n_test, n_features, device=dev, generator=g)
        self.y_test = yt
        self.counts = counts

    def federation(self, test_slice: tuple[int, int] | None = None):
        from .experiment import DeviceFederation
        xt, yt = self.x_test, self.y_test
        if test_slice is not None:
            xt, yt = xt[test_slice[0]:test_slice[1]].contiguous(), yt[test_slice[0]:test_slice[1]].contiguous()
        return DeviceFederation.from_arrays(self.x, self.y, self.offsets, xt, yt, self.n_classes)
