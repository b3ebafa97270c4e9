"""Client sharding across GPUs (one process per GPU) and the FedAvg exchange.

A round's participants are independent given the round-start model
(engine.py:336-347), so they shard over ranks with no data-path traffic
(longest-processing-time on each client's row count, `lpt_shards`); the one
exchange step is the sum in FedAvg (fl_core.py:215-217):

    S_r = sum_{i in shard r} (w_i / W) * delta_i        (fp64, fedavg_kernel, base = NULL)
    S   = all_reduce_sum(S_r)                           (NCCL over NVLink/NVSwitch)
    params <- params + S                                (fedavg_kernel, K = 1, coef = 1)

W is the GLOBAL sample total, known on every rank from the (replicated,
deterministic) selection.  Test-set accuracy shards by rows and all-reduces
an int64 count.  The arithmetic differs from the reference's sequential
fp64 loop only in summation order (fp64, ~1e-16 relative).
"""

from __future__ import annotations

import torch


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous balanced slice [lo, hi) of n items for `rank` (first n % world ranks get one more)."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def lpt_shards(costs, world: int) -> list[list[int]]:
    """Longest-processing-time assignment of items to `world` ranks.

    Items in decreasing cost (ties: lower index first) go to the currently least-loaded rank (ties: lower
    rank).  Deterministic, so every rank computes the same assignment from the replicated selection.
    Each rank's list is returned in increasing item index (= selection order), so a rank trains and sums
    its clients in the reference's list order.
    """
    if world < 1:
        raise ValueError("world must be >= 1")
    import heapq

    order = sorted(range(len(costs)), key=lambda i: (-float(costs[i]), i))
    heap = [(0.0, r) for r in range(world)]
    out: list[list[int]] = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        out[r].append(i)
        heapq.heappush(heap, (load + float(costs[i]), r))
    for lst in out:
        lst.sort()
    return out


def client_cost(num_samples: int, batch_size: int, n_rows: int | None = None) -> float:
    """GPU cost of one client's local_train: rows it processes (fl_core.py:180-189: ceil(n/B) batches
    of B rows; a shard smaller than its workload reshuffles, so the row count is the workload's)."""
    if n_rows == 0 or num_samples <= 0:
        return 0.0
    return float(-(-int(num_samples) // int(batch_size)) * int(batch_size))


def shard_participants(participants: list[str], world: int, rank: int) -> list[str]:
    lo, hi = shard_bounds(len(participants), world, rank)
    return participants[lo:hi]


def global_coefficients(weights_all: list[float], lo: int, hi: int) -> list[float]:
    """Coefficients w_i / W for this shard, W = float(sum(all weights)) as in fl_core.py:207."""
    total = float(sum(weights_all))
    return [w / total for w in weights_all[lo:hi]]


def combine_partials(partial: torch.Tensor, params: torch.Tensor, apply_fn, group=None) -> torch.Tensor:
    """All-reduce the per-rank partial FedAvg sums, then params <- params + S via `apply_fn`.

    `apply_fn(S, params)` is the device FedAvg apply (fedavg_kernel with K = 1) on GPU ranks and a
    plain add in CPU (gloo) tests.
    """
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(partial, group=group)
    return apply_fn(partial, params)


def all_reduce_count(count: torch.Tensor, group=None) -> torch.Tensor:
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(count, group=group)
    return count
