"""N > 1 path on CPU: world_size-2 gloo processes run the sharded round
(participant sharding, per-rank partial FedAvg sums, all-reduce, apply,
sharded accuracy count) with the oracle standing in for the GPU kernels, and
must reproduce the single-process reference round."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2305_15668_b200.sharding import (all_reduce_count, combine_partials, global_coefficients, shard_bounds,
                                            shard_participants)


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_bounds_cover_exactly_once():
    for n in range(0, 40):
        for world in range(1, 9):
            seen = []
            for r in range(world):
                lo, hi = shard_bounds(n, world, r)
                seen += list(range(lo, hi))
                assert hi - lo in (n // world, n // world + 1)
            assert seen == list(range(n))


def _worker(rank, world, port, out_path):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import flmath as fm
    from oracle import orchestration as oc

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    fleet = oc.fleet(9, 3, budget_levels=(10, 30, 50), num_samples=[96, 128, 150], batch_size=[32, 50])
    by_id = {c.client_id: c for c in fleet}
    F, C = 6, 4
    tr, test = fm.synthetic(F, C, 2000, seed=7)
    shards = fm.dirichlet_partition(tr, [(c.client_id, c.workload.num_samples) for c in fleet], 0.5, seed=8)
    params = np.random.default_rng(0).standard_normal(F * C + C) * 0.1
    import random
    who = random.Random("3:selection").sample(sorted(by_id), 7)
    mine = shard_participants(who, world, rank)
    lo, hi = shard_bounds(len(who), world, rank)
    weights = [float(by_id[c].workload.num_samples) for c in who]
    coef = global_coefficients(weights, lo, hi)
    partial = np.zeros_like(params)
    for c, k in zip(mine, coef):
        wl = by_id[c].workload
        d = fm.local_sgd(params, shards[c], wl.num_samples, wl.batch_size, 0.1, C, seed=fm.seed_of("train", 3, 0, c))
        partial = partial + k * d
    out = combine_partials(torch.from_numpy(partial), torch.from_numpy(params), lambda s, p: p + s)
    # sharded accuracy
    tlo, thi = shard_bounds(len(test.labels), world, rank)
    W, b = fm.split_params(out.numpy(), F, C)
    pred = np.argmax(test.features[tlo:thi] @ W + b, axis=1)
    cnt = all_reduce_count(torch.tensor([int(np.sum(pred == test.labels[tlo:thi]))], dtype=torch.int64))
    if rank == 0:
        np.savez(out_path, params=out.numpy(), correct=cnt.numpy(), who=np.array(who))
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_round_matches_single_process(tmp_path):
    from oracle import flmath as fm
    from oracle import orchestration as oc

    out_path = str(tmp_path / "rank0.npz")
    mp.start_processes(_worker, args=(2, free_port(), out_path), nprocs=2, join=True, start_method="spawn")
    got = np.load(out_path)
    # single-process reference round
    fleet = oc.fleet(9, 3, budget_levels=(10, 30, 50), num_samples=[96, 128, 150], batch_size=[32, 50])
    by_id = {c.client_id: c for c in fleet}
    F, C = 6, 4
    tr, test = fm.synthetic(F, C, 2000, seed=7)
    shards = fm.dirichlet_partition(tr, [(c.client_id, c.workload.num_samples) for c in fleet], 0.5, seed=8)
    params = np.random.default_rng(0).standard_normal(F * C + C) * 0.1
    who = [str(c) for c in got["who"]]  # np.str_ would change repr() and so stable_seed
    deltas = [fm.local_sgd(params, shards[c], by_id[c].workload.num_samples, by_id[c].workload.batch_size, 0.1, C,
                           seed=fm.seed_of("train", 3, 0, c)) for c in who]
    want = fm.weighted_average(deltas, [float(by_id[c].workload.num_samples) for c in who], params)
    assert np.max(np.abs(got["params"] - want)) <= 1e-12 * np.max(np.abs(want))
    assert int(got["correct"][0]) == round(fm.accuracy(want, test) * len(test.labels))



def test_lpt_shards_balance_heterogeneous_round():
    """The LPT split of a config-4-like round (sample counts 16..1024) is within one client's cost of the
    average load, where contiguous slices are not."""
    import random
    from paper_2305_15668_b200.sharding import client_cost, lpt_shards, shard_bounds
    rng = random.Random(0)
    costs = [client_cost(rng.choice([16, 32, 64, 128, 256, 512, 1024]), 32) for _ in range(200)]
    for world in (2, 4, 8):
        shards = lpt_shards(costs, world)
        loads = [sum(costs[i] for i in s) for s in shards]
        assert max(loads) - min(loads) <= max(costs)
        contiguous = [sum(costs[slice(*shard_bounds(len(costs), world, r))]) for r in range(world)]
        assert max(loads) <= max(contiguous)


def test_lpt_shards_cover_exactly_once_and_keep_selection_order():
    from paper_2305_15668_b200.sharding import lpt_shards
    rng = np.random.default_rng(1)
    for n in range(0, 30):
        costs = rng.integers(0, 5, n).tolist()
        for world in range(1, 6):
            shards = lpt_shards(costs, world)
            flat = sorted(i for s in shards for i in s)
            assert flat == list(range(n))
            assert all(s == sorted(s) for s in shards)
            assert shards == lpt_shards(costs, world)   # deterministic on every rank
    # uniform costs: equal counts
    assert [len(s) for s in lpt_shards([64.0] * 200, 8)] == [25] * 8
