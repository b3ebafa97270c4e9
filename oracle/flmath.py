"""Oracle restatement of the reference FL math (TEST INFRASTRUCTURE ONLY).

Every function cites the reference line range it restates
(``pkg/src/fedsim/fl_core.py`` in /root/reference).  The arithmetic is fp64
numpy, in the same operation order as the reference, and the random draws are
issued in exactly the same sequence so that datasets, partitions and batch
orders are bit-identical to the reference for the same seed.
"""

from __future__ import annotations

import hashlib
import math
from typing import NamedTuple

import numpy as np


class AggregationError(Exception):
    """Mirrors fedsim.errors.AggregationError (errors.py:12-13)."""


class Data(NamedTuple):
    """(features [n,F] f64, labels [n] int, n_classes) -- fl_core.py:27-31."""

    features: np.ndarray
    labels: np.ndarray
    num_classes: int


class Shard(NamedTuple):
    """One client's rows -- fl_core.py:34-38."""

    owner: str
    features: np.ndarray
    labels: np.ndarray


def seed_of(*parts) -> int:
    """fl_core.py:21-24: first 4 bytes (LE) of sha256(repr(parts))."""
    return int.from_bytes(hashlib.sha256(repr(parts).encode()).digest()[:4], "little")


def synthetic(n_features: int, n_classes: int, n_total: int, seed: int):
    """fl_core.py:41-59: Gaussian clusters, returns (train, test)."""
    if n_features < 1 or n_classes < 2:
        raise ValueError("need n_features >= 1 and n_classes >= 2")
    gen = np.random.default_rng(seed)
    centers = 3.0 * gen.standard_normal((n_classes, n_features))
    if n_total == 0:
        blank = lambda: Data(np.zeros((0, n_features)), np.zeros(0, dtype=int), n_classes)
        return blank(), blank()
    y = gen.integers(0, n_classes, size=n_total)
    x = centers[y] + gen.standard_normal((n_total, n_features))
    cut = n_total // 5
    return Data(x[cut:], y[cut:], n_classes), Data(x[:cut], y[:cut], n_classes)


def dirichlet_partition(data: Data, clients, alpha: float, seed: int) -> dict:
    """fl_core.py:62-115: per-client Dirichlet class mix, drawn without replacement."""
    if alpha <= 0:
        raise ValueError("alpha must be > 0")
    need = sum(k for _, k in clients)
    if need > len(data.labels):
        raise ValueError(f"clients want {need} samples but dataset has {len(data.labels)}")
    gen = np.random.default_rng(seed)
    C = data.num_classes
    pool = []
    for c in range(C):
        members = list(np.flatnonzero(data.labels == c))
        gen.shuffle(members)
        pool.append(members)
    out = {}
    for owner, k in clients:
        mix = gen.dirichlet([alpha] * C)
        quota = np.floor(mix * k).astype(int)
        leftover = k - quota.sum()
        # largest fractional parts get the integer remainder (stable order)
        bump = np.argsort(-(mix * k - quota), kind="stable")[:leftover]
        for c in bump:
            quota[c] += 1
        picked: list[int] = []
        deficit = 0
        for c in range(C):
            got = min(quota[c], len(pool[c]))
            deficit += quota[c] - got
            if got:
                picked.extend(pool[c][-got:])
                del pool[c][-got:]
        while deficit > 0:
            sizes = [len(p) for p in pool]
            best = sizes.index(max(sizes))  # first class with the most rows left
            if not pool[best]:
                raise ValueError("dataset exhausted during partitioning")
            picked.append(pool[best].pop())
            deficit -= 1
        rows = np.array(sorted(picked), dtype=int)
        out[owner] = Shard(owner, data.features[rows], data.labels[rows])
    return out


# -- multinomial logistic regression (fl_core.py:118-160) -------------------


def zeros_params(n_features: int, n_classes: int) -> np.ndarray:
    """fl_core.py:121-123: [W (F x C, row-major) ; b (C)] all zero."""
    return np.zeros(n_features * n_classes + n_classes)


def split_params(theta: np.ndarray, n_features: int, n_classes: int):
    """fl_core.py:126-129."""
    cut = n_features * n_classes
    return theta[:cut].reshape(n_features, n_classes), theta[cut:]


def ce_grad(theta: np.ndarray, x: np.ndarray, y: np.ndarray, n_classes: int):
    """fl_core.py:132-151: mean CE loss and flat gradient [gW ; gb]."""
    rows, feats = x.shape
    W, b = split_params(theta, feats, n_classes)
    z = x @ W + b
    z = z - z.max(axis=1, keepdims=True)
    p = np.exp(z)
    p = p / p.sum(axis=1, keepdims=True)
    pick = np.arange(rows)
    loss = -float(np.mean(np.log(p[pick, y] + 1e-300)))
    p[pick, y] -= 1.0
    p /= rows
    return loss, np.concatenate([(x.T @ p).ravel(), p.sum(axis=0)])


def accuracy(theta: np.ndarray, data: Data) -> float:
    """fl_core.py:154-160: first-max argmax accuracy."""
    if len(data.labels) == 0:
        return 0.0
    W, b = split_params(theta, data.features.shape[1], data.num_classes)
    return float(np.mean(np.argmax(data.features @ W + b, axis=1) == data.labels))


def batch_plan(n_rows: int, num_samples: int, batch_size: int, seed) -> list[np.ndarray]:
    """The row order local_train visits (fl_core.py:176-189).

    ceil(num_samples / batch_size) batches; a fresh PCG64 permutation each
    time the shard is exhausted; the batch before a reshuffle may be ragged.
    """
    if n_rows == 0:
        return []
    gen = np.random.default_rng(seed_of("local_train", seed))
    perm = gen.permutation(n_rows)
    at = 0
    plan = []
    for _ in range(math.ceil(num_samples / batch_size)):
        if at >= n_rows:
            perm = gen.permutation(n_rows)
            at = 0
        plan.append(perm[at : at + batch_size])
        at += batch_size
    return plan


def local_sgd(theta, shard: Shard, num_samples: int, batch_size: int, lr: float,
              n_classes: int, seed=0) -> np.ndarray:
    """fl_core.py:163-194: mini-batch SGD from theta; returns the delta."""
    w = theta.copy()
    for rows in batch_plan(len(shard.labels), num_samples, batch_size, seed):
        _, g = ce_grad(w, shard.features[rows], shard.labels[rows], n_classes)
        w -= lr * g
    return w - theta


def weighted_average(deltas, weights, base: np.ndarray) -> np.ndarray:
    """fl_core.py:197-218: base + sum_i (w_i / sum w) * delta_i, in list order."""
    if not deltas:
        raise AggregationError("no deltas to aggregate")
    if len(deltas) != len(weights):
        raise AggregationError("deltas and weights length mismatch")
    if any(w < 0 for w in weights):
        raise AggregationError("weights must be non-negative")
    total = float(sum(weights))
    if total == 0:
        raise AggregationError("weights must not all be zero")
    for d in deltas:
        if d.shape != base.shape:
            raise AggregationError(f"delta shape {d.shape} does not match base {base.shape}")
    acc = base.copy()
    for d, w in zip(deltas, weights):
        acc += (w / total) * d
    return acc
