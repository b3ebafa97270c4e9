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
Values of DeviceFleetData are NOT bit-identical to the reference (its class
quotas are, the values are drawn by torch's generator).

reference_federation() is the bit-identical variant: the class centres and
labels are drawn on the host from the reference's own PCG64 stream (cheap:
C*F + n draws), the n*F feature noise -- the bulk of the work -- is generated
on the device by fedhc_pcg64_standard_normal, which reproduces numpy's
Generator.standard_normal (ziggurat over PCG64) draw for draw by splitting the
stream into fixed runs of raw outputs and chaining the per-run acceptance
counts, and the partition is the reference's own pool bookkeeping on the host
labels (training.partition_rows).  Its tensors equal
DeviceFederation(partition_noniid(make_synthetic_dataset(...))) bit for bit.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _abi
from .training import device, partition_rows, stream_ptr

_M64 = (1 << 64) - 1


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


def pcg64_standard_normal(state: dict, n: int, out: torch.Tensor | None = None) -> tuple[torch.Tensor, dict]:
    """numpy ``Generator(PCG64).standard_normal(n)`` from bit-generator state ``state``, on the device.

    ``state`` is ``rng.bit_generator.state`` of the reference's generator (fl_core.py:44-55 draws
    through numpy's ziggurat, distributions.c random_standard_normal).  Returns the fp64 normals
    [n] on the current device and the bit-generator state after them (what
    ``rng.bit_generator.state`` would read after ``rng.standard_normal(n)``).
    """
    if state.get("bit_generator") != "PCG64":
        raise ValueError("standard_normal: only PCG64 streams are supported")
    s, inc = int(state["state"]["state"]), int(state["state"]["inc"])
    words = np.array([s >> 64, s & _M64, inc >> 64, inc & _M64], dtype=np.uint64)
    after = np.zeros(2, dtype=np.uint64)
    if out is None:
        out = torch.empty(n, dtype=torch.float64, device=device())
    if out.dtype != torch.float64 or not out.is_contiguous() or out.numel() < n:
        raise ValueError("standard_normal: out must be contiguous fp64 with >= n elements")
    _abi.check(_abi.lib.fedhc_pcg64_standard_normal(words.ctypes.data, int(n), out.data_ptr(),
                                                     after.ctypes.data, stream_ptr()))
    new = {"bit_generator": "PCG64",
           "state": {"state": (int(after[0]) << 64) | int(after[1]), "inc": inc},
           "has_uint32": state.get("has_uint32", 0), "uinteger": state.get("uinteger", 0)}
    return out[:n], new


def synthetic_dataset(n_features: int, n_classes: int, n_total: int, seed: int, chunk_rows: int = 1 << 18):
    """make_synthetic_dataset (fl_core.py:41-59) with the features produced in HBM.

    Returns device tensors (x fp32 [n_total, F] = fp32(centers[y] + noise) computed in fp64 like the
    reference, y int32 [n_total]) plus the host labels; rows [0, n_total // 5) are the test split.
    """
    if n_features < 1 or n_classes < 2:
        raise ValueError("need n_features >= 1 and n_classes >= 2")
    dev = device()
    rng = np.random.default_rng(seed)
    centers = torch.from_numpy(rng.standard_normal((n_classes, n_features)) * 3.0).to(dev)
    y_host = rng.integers(0, n_classes, size=n_total) if n_total else np.zeros(0, dtype=np.int64)
    y = torch.from_numpy(y_host).to(dev)
    x = torch.empty(n_total, n_features, dtype=torch.float32, device=dev)
    state = rng.bit_generator.state
    rows = max(1, min(chunk_rows, n_total))
    noise = torch.empty(rows * n_features, dtype=torch.float64, device=dev)
    for a in range(0, n_total, rows):
        b = min(a + rows, n_total)
        z, state = pcg64_standard_normal(state, (b - a) * n_features, noise)
        x[a:b] = (centers[y[a:b]] + z.view(b - a, n_features)).to(torch.float32)
    return x, y.to(torch.int32), y_host


def reference_federation(clients: list[tuple[str, int]], n_features: int, n_classes: int, n_total: int,
                         data_seed: int, alpha: float, partition_seed: int):
    """The reference experiment's data (fl_core.py:41-115) built in HBM, bit-identical.

    Equals ``DeviceFederation(partition_noniid(train, clients, alpha, partition_seed), test, F, C)``
    with ``train, test = make_synthetic_dataset(F, C, n_total, data_seed)``, without materialising
    the fp64 dataset on the host.
    """
    from .experiment import DeviceFederation
    x, y, y_host = synthetic_dataset(n_features, n_classes, n_total, data_seed)
    n_test = n_total // 5
    rows = partition_rows(y_host[n_test:], n_classes, clients, alpha, partition_seed)
    offsets, at, parts = {}, 0, []
    for cid, _ in clients:
        sel = rows[cid]
        offsets[cid] = (at, len(sel))
        at += len(sel)
        parts.append(sel + n_test)
    order = torch.from_numpy(np.concatenate(parts) if parts else np.zeros(0, dtype=np.int64)).to(x.device)
    if at == 0:                                   # DeviceFederation keeps one zero row for an empty fleet
        xs = torch.zeros(1, n_features, device=x.device)
        ys = torch.zeros(1, dtype=torch.int32, device=x.device)
    else:
        xs, ys = x[order].contiguous(), y[order].contiguous()
    return DeviceFederation.from_arrays(xs, ys, offsets, x[:n_test].contiguous(), y[:n_test].contiguous(),
                                        n_classes)
