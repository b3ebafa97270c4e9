"""N > 1 through the product round path: two ranks of `FederatedRunner` (world = 2)
share cuda:0 over the gloo backend (CUDA tensors) -- LPT participant shards,
per-rank partial FedAvg sums (fedavg_kernel, base = NULL), the all-reduce, the
apply, the sharded accuracy count -- and must reproduce the world = 1 run of
the same rounds (engine.py:326-353 sync semantics): params within 1e-12
relative (fp64 summation order is the only difference) and the per-round
accuracy series exactly."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROUNDS = 3


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _setup(aggregation="sync"):
    import torch
    import paper_2305_15668_b200 as fh
    from paper_2305_15668_b200.devicedata import DeviceFleetData
    torch.cuda.set_device(0)
    # heterogeneous sample counts and batch sizes: LPT gives the ranks different client counts
    fleet = fh.generate_fleet(fh.DistributionSpec(budget_levels=(10, 30, 50, 80), num_samples=[192, 640, 704],
                                                  batch_size=[32, 64]), 30, 11)
    by_id = {p.client_id: p for p in fleet}
    ids = sorted(by_id)
    data = DeviceFleetData(ids, [by_id[c].workload.num_samples for c in ids], 784, 10, 0.5, seed=5, n_test=1999)
    cfg = fh.FleetConfig(participants_per_round=17, max_executors=8, seed=11, aggregation=aggregation,
                         async_buffer=4)
    return fh, by_id, data, cfg


def _worker(rank, world, port, out_dir, aggregation):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    from paper_2305_15668_b200.experiment import FederatedRunner

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    fh, by_id, data, cfg = _setup(aggregation)
    params = torch.zeros(7850, dtype=torch.float64, device="cuda")
    runner = FederatedRunner(data.federation(), by_id, cfg, 0.1, params=params, world=world, rank=rank)
    series = runner.run(ROUNDS)
    plans_k = len(runner.deltas)
    torch.cuda.synchronize()
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), params=params.cpu().numpy(), series=np.array(series),
             k=plans_k)
    dist.destroy_process_group()


@pytest.mark.timeout(600)
@pytest.mark.parametrize("aggregation", ["sync", "async"])
def test_two_rank_runner_matches_single_rank(tmp_path, aggregation):
    """Sync: one all-reduce per round.  Async (engine.py:354-364, async_buffer 4): one all-reduce of the chunk's
    partial sums and one sharded accuracy per chunk; the world = 1 run is the native round loop."""
    import torch
    import torch.multiprocessing as mp
    from paper_2305_15668_b200.experiment import FederatedRunner

    fh, by_id, data, cfg = _setup(aggregation)
    params = torch.zeros(7850, dtype=torch.float64, device="cuda")
    runner = FederatedRunner(data.federation(), by_id, cfg, 0.1, params=params)
    assert runner._native is not None
    want_series = runner.run(ROUNDS)
    want = params.cpu().numpy()
    if aggregation == "async":
        assert len(want_series) == ROUNDS * 5  # ceil(17 / 4) chunks per round

    mp.start_processes(_worker, args=(2, free_port(), str(tmp_path), aggregation), nprocs=2, join=True,
                       start_method="spawn")
    for rank in range(2):
        got = np.load(tmp_path / f"rank{rank}.npz")
        assert np.max(np.abs(got["params"] - want)) <= 1e-12 * np.max(np.abs(want))
        assert [tuple(x) for x in got["series"].tolist()] == [tuple(x) for x in want_series]

