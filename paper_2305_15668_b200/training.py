"""FL math API on the B200 -- drop-in for fedsim.fl_core (fl_core.py:1-218).

Host side (setup, bit-identical to the reference for the same seed):
  stable_seed, Dataset/DatasetShard, make_synthetic_dataset, partition_noniid,
  init_params, batch_permutations (the PCG64 batch order of local_train).
Device side (libfedhc kernels, no CPU fallback):
  local_train  -> fedhc_local_train   (fused SGD, bf16x3 tensor-core products, fp32 state)
  fedavg       -> fedhc_fedavg        (fp64, bit-identical for fp64 deltas)
  evaluate_accuracy -> fedhc_eval
  loss_and_grad -> fedhc_loss_and_grad (fp64)
The numpy-in / numpy-out functions copy to and from the GPU on every call;
the batched, HBM-resident round path lives in `experiment.DeviceFederation`.
"""

from __future__ import annotations

import ctypes as C
import hashlib
import math
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _abi
from .errors import AggregationError


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2305_15668_b200 needs a CUDA device (B200, sm_100a); no CPU fallback exists")
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def stable_seed(*parts) -> int:
    """32-bit seed from sha256(repr(parts)) (fl_core.py:21-24)."""
    return int.from_bytes(hashlib.sha256(repr(parts).encode()).digest()[:4], "little")


@dataclass
class Dataset:
    features: np.ndarray
    labels: np.ndarray
    num_classes: int


@dataclass
class DatasetShard:
    owner: str
    features: np.ndarray
    labels: np.ndarray


def make_synthetic_dataset(n_features: int, n_classes: int, n_total: int, seed: int) -> tuple[Dataset, Dataset]:
    """Gaussian class clusters, 20% held out (fl_core.py:41-59; same PCG64 draws)."""
    if n_features < 1 or n_classes < 2:
        raise ValueError("need n_features >= 1 and n_classes >= 2")
    rng = np.random.default_rng(seed)
    centers = rng.standard_normal((n_classes, n_features)) * 3.0
    if n_total == 0:
        return (Dataset(np.zeros((0, n_features)), np.zeros(0, dtype=int), n_classes),
                Dataset(np.zeros((0, n_features)), np.zeros(0, dtype=int), n_classes))
    y = rng.integers(0, n_classes, size=n_total)
    x = centers[y] + rng.standard_normal((n_total, n_features))
    n_test = n_total // 5
    return Dataset(x[n_test:], y[n_test:], n_classes), Dataset(x[:n_test], y[:n_test], n_classes)


def partition_rows(labels: np.ndarray, n_classes: int, clients: list[tuple[str, int]], alpha: float,
                   seed: int) -> dict[str, np.ndarray]:
    """Row indices of each client's shard: the draws and pool bookkeeping of fl_core.py:62-115.

    Per-class pools are shuffled once (same PCG64 draws for an ndarray as for the
    reference's list), each client takes floor(Dir(alpha) * n) rows per class plus
    the largest-remainder fix-up from the pool tails, any shortfall comes from the
    first richest pool, and the shard's rows are sorted ascending.
    """
    if alpha <= 0:
        raise ValueError("alpha must be > 0")
    wanted = sum(n for _, n in clients)
    if wanted > len(labels):
        raise ValueError(f"clients want {wanted} samples but dataset has {len(labels)}")
    rng = np.random.default_rng(seed)
    pools = []
    for c in range(n_classes):
        members = np.flatnonzero(labels == c)
        rng.shuffle(members)
        pools.append(members)
    live = [len(p) for p in pools]          # pools[c][:live[c]] is what is left of class c
    out: dict[str, np.ndarray] = {}
    for cid, n in clients:
        mix = rng.dirichlet([alpha] * n_classes)
        counts = np.floor(mix * n).astype(int)
        extra = n - counts.sum()
        for c in np.argsort(-(mix * n - counts), kind="stable")[:extra]:
            counts[c] += 1
        parts: list[np.ndarray] = []
        short = 0
        for c in range(n_classes):
            take = int(min(counts[c], live[c]))
            short += int(counts[c]) - take
            if take:
                parts.append(pools[c][live[c] - take:live[c]])
                live[c] -= take
        for _ in range(short):
            richest = live.index(max(live))
            if not live[richest]:
                raise ValueError("dataset exhausted during partitioning")
            live[richest] -= 1
            parts.append(pools[richest][live[richest]:live[richest] + 1])
        out[cid] = np.sort(np.concatenate(parts)) if parts else np.zeros(0, dtype=int)
    return out


def partition_noniid(dataset: Dataset, clients: list[tuple[str, int]], alpha: float,
                     seed: int) -> dict[str, DatasetShard]:
    """Dirichlet(alpha) label mix per client, drawn without replacement (fl_core.py:62-115)."""
    rows = partition_rows(dataset.labels, dataset.num_classes, clients, alpha, seed)
    return {cid: DatasetShard(cid, dataset.features[sel], dataset.labels[sel]) for cid, sel in rows.items()}


def init_params(n_features: int, n_classes: int) -> np.ndarray:
    return np.zeros(n_features * n_classes + n_classes)


def n_permutations(n_rows: int, num_samples: int, batch_size: int) -> int:
    """How many epochs' permutations local_train consumes (fl_core.py:180-187)."""
    if n_rows == 0:
        return 0
    steps = math.ceil(num_samples / batch_size)
    per_epoch = math.ceil(n_rows / batch_size)
    return max(1, math.ceil(steps / per_epoch))


def native_permutations(seeds, n_rows, n_perms, out: np.ndarray | None = None, threads: int = 0) -> np.ndarray:
    """Native (libfedhc, multi-threaded) PCG64 permutations, bit-exact with numpy.

    seeds[c] is the default_rng seed (stable_seed("local_train", seed)); client c
    gets n_perms[c] concatenated permutations of range(n_rows[c]).
    """
    seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
    rows = np.ascontiguousarray(n_rows, dtype=np.int32)
    perms = np.ascontiguousarray(n_perms, dtype=np.int32)
    sizes = rows.astype(np.int64) * perms
    offsets = np.zeros(len(sizes), dtype=np.int64)
    if len(sizes) > 1:
        np.cumsum(sizes[:-1], out=offsets[1:])
    total = int(sizes.sum())
    if out is None:
        out = np.empty(total, dtype=np.int32)
    assert out.dtype == np.int32 and out.flags.c_contiguous and out.shape[0] >= total
    _abi.check(_abi.lib.fedhc_batch_permutations(seeds.ctypes.data, rows.ctypes.data, perms.ctypes.data,
                                                 offsets.ctypes.data, len(seeds), out.ctypes.data, threads))
    return out[:total]


def batch_permutations(n_rows: int, num_samples: int, batch_size: int, seed) -> np.ndarray:
    """Concatenated PCG64 permutations that local_train's batches walk (int32)."""
    k = n_permutations(n_rows, num_samples, batch_size)
    if k == 0:
        return np.zeros(0, dtype=np.int32)
    return native_permutations([stable_seed("local_train", seed)], [n_rows], [k])


def _dev_array(a: np.ndarray, dtype) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a, dtype=dtype)).to(device())


def descriptors_to_device(descs) -> torch.Tensor:
    raw = bytearray(descs)
    return torch.frombuffer(raw, dtype=torch.uint8).to(device())


def loss_and_grad(params: np.ndarray, features: np.ndarray, labels: np.ndarray, n_classes: int):
    """Mean cross-entropy and analytic gradient, fp64 on the GPU (fl_core.py:138-151)."""
    n, n_features = features.shape
    x = _dev_array(features, np.float64)
    y = _dev_array(labels, np.int32)
    p = _dev_array(params, np.float64)
    grad = torch.empty_like(p)
    loss = torch.empty(1, dtype=torch.float64, device=p.device)
    ws = torch.empty(n * n_classes, dtype=torch.float64, device=p.device)
    _abi.check(_abi.lib.fedhc_loss_and_grad(x.data_ptr(), y.data_ptr(), n, n_features, n_classes, p.data_ptr(),
                                            grad.data_ptr(), loss.data_ptr(), ws.data_ptr(), stream_ptr()))
    return float(loss.item()), grad.cpu().numpy()


def evaluate_accuracy(params: np.ndarray, dataset: Dataset) -> float:
    """Fraction of rows whose first-max argmax equals the label (fl_core.py:154-160)."""
    n = len(dataset.labels)
    if n == 0:
        return 0.0
    x = _dev_array(dataset.features, np.float32)
    y = _dev_array(dataset.labels, np.int32)
    p = _dev_array(params, np.float64)
    return count_correct(x, y, p, dataset.num_classes) / n


def count_correct(x: torch.Tensor, y: torch.Tensor, params: torch.Tensor, n_classes: int) -> int:
    correct = torch.zeros(1, dtype=torch.int64, device=x.device)
    _abi.check(_abi.lib.fedhc_eval(x.data_ptr(), y.data_ptr(), x.shape[0], x.shape[1], n_classes,
                                   params.data_ptr(), correct.data_ptr(), stream_ptr()))
    return int(correct.item())


def train_sms_per_client(n_features: int, n_classes: int) -> int:
    """SMs one client's local SGD occupies in fedhc_local_train's dispatch (csrc/train.cu local_train_impl):
    the one-CTA trainers (F <= 784, C <= 16), 2-CTA clusters (16 < C <= 64 at F <= 784: train_fused /
    train_c64_kernel), the F-split tcgen05 clusters of train_tc_kernel above F = 784 (4 or 8 CTAs; 8 taken as
    the bound).  The round loop sizes its side-work SM windows from this."""
    if n_features <= 784:
        return 1 if n_classes <= 16 else 2
    return 8


def split_supported(n_features: int, n_classes: int) -> bool:
    """Shapes whose trainer reads the fedhc_x_split row copy: the one-CTA mma.sync trainer (F = 784, C <= 16)
    and the tcgen05 cluster trainer (F > 784 or 32 < C <= 64, F % 8 == 0).  FEDHC_X_SPLIT=0 keeps every launch
    on the fp32 rows (A/B measurements)."""
    if os.environ.get("FEDHC_X_SPLIT", "1") == "0":
        return False
    if n_features == 784 and n_classes <= 16:
        return True
    return (n_features > 784 or 32 < n_classes <= 64) and n_features % 8 == 0 and n_classes <= 64


def x_split(x: torch.Tensor) -> torch.Tensor:
    """The rows of x (fp32 [n, F], device) re-encoded per 8-feature unit as [8 bf16 hi | 8 bf16 mid]: same
    bytes, so the copy is returned as an opaque fp32-typed tensor of x's shape (fedhc_x_split)."""
    out = torch.empty_like(x)
    _abi.check(_abi.lib.fedhc_x_split(x.data_ptr(), int(x.shape[0]), int(x.shape[1]), out.data_ptr(), stream_ptr()))
    return out


def train_launch(desc_ptr: int, k: int, params_ptr: int, n_features: int, n_classes: int, max_batch: int,
                 x: torch.Tensor | None = None, xs: torch.Tensor | None = None, stream: int | None = None) -> None:
    """One fedhc_local_train launch for k device descriptors; with a split copy xs of the rows x the
    descriptors point into, the launch reads the copy where a kernel for it exists (bit-identical results)."""
    st = stream_ptr() if stream is None else stream
    if xs is not None:
        _abi.check(_abi.lib.fedhc_local_train_split(desc_ptr, k, params_ptr, n_features, n_classes, max_batch,
                                                    xs.data_ptr() - x.data_ptr(), st))
    else:
        _abi.check(_abi.lib.fedhc_local_train(desc_ptr, k, params_ptr, n_features, n_classes, max_batch, st))


def local_train(params: np.ndarray, shard: DatasetShard, workload, lr: float, n_classes: int,
                seed: int | str = 0) -> np.ndarray:
    """Mini-batch SGD on one client's shard; returns the delta (fl_core.py:163-194)."""
    n = len(shard.labels)
    if n == 0:
        return params.copy() - params
    n_features = shard.features.shape[1]
    x = _dev_array(shard.features, np.float32)
    y = _dev_array(shard.labels, np.int32)
    perm = _dev_array(batch_permutations(n, workload.num_samples, workload.batch_size, seed), np.int32)
    p = _dev_array(params, np.float64)
    delta = torch.empty(p.shape[0], dtype=torch.float32, device=p.device)
    desc = (_abi.Client * 1)(_abi.Client(x.data_ptr(), y.data_ptr(), perm.data_ptr(), n,
                                         math.ceil(workload.num_samples / workload.batch_size),
                                         workload.batch_size, float(lr), delta.data_ptr()))
    d_desc = descriptors_to_device(desc)
    xs = x_split(x) if split_supported(n_features, n_classes) else None
    train_launch(d_desc.data_ptr(), 1, p.data_ptr(), n_features, n_classes, workload.batch_size, x, xs)
    return delta.cpu().numpy().astype(np.float64)


def check_aggregation(deltas, weights, base_shape) -> float:
    """fl_core.py:201-214 validation; returns total = float(sum(weights))."""
    if not len(deltas):
        raise AggregationError("no deltas to aggregate")
    if len(deltas) != len(weights):
        raise AggregationError("deltas and weights length mismatch")
    if any(w < 0 for w in weights):
        raise AggregationError("weights must be non-negative")
    total = float(sum(weights))
    if total == 0:
        raise AggregationError("weights must not all be zero")
    for d in deltas:
        if tuple(d.shape) != tuple(base_shape):
            raise AggregationError(f"delta shape {tuple(d.shape)} does not match base {tuple(base_shape)}")
    return total


def fedavg_device(deltas: torch.Tensor, coef: torch.Tensor, base: torch.Tensor | None, out: torch.Tensor,
                  rows: torch.Tensor | None = None) -> torch.Tensor:
    """out = base + sum_k coef[k] * deltas[k] on the GPU (packed [K, P] or pointer rows)."""
    dtype = _abi.F32 if deltas.dtype == torch.float32 else _abi.F64
    n = out.shape[0]
    k = coef.shape[0]
    _abi.check(_abi.lib.fedhc_fedavg(rows.data_ptr() if rows is not None else None,
                                     deltas.data_ptr() if rows is None else None, deltas.stride(0) if rows is None
                                     else 0, dtype, coef.data_ptr(), k,
                                     base.data_ptr() if base is not None else None, out.data_ptr(), n,
                                     stream_ptr()))
    return out


def fedavg(deltas: list[np.ndarray], weights: list[float], base: np.ndarray) -> np.ndarray:
    """base + sample-weighted mean of deltas, fp64, list order (fl_core.py:197-218)."""
    total = check_aggregation(deltas, weights, base.shape)
    coef = _dev_array(np.array([w / total for w in weights], dtype=np.float64), np.float64)
    stack = _dev_array(np.stack([np.asarray(d, dtype=np.float64).reshape(-1) for d in deltas]), np.float64)
    b = _dev_array(base.reshape(-1), np.float64)
    out = torch.empty_like(b)
    fedavg_device(stack, coef, b, out)
    return out.cpu().numpy().reshape(base.shape)
