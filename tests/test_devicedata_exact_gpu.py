"""On-device numpy-exact synthetic data.

fedhc_pcg64_standard_normal must reproduce numpy's Generator.standard_normal
(ziggurat over PCG64, the draws behind fl_core.py:47-55) draw for draw, and
reference_federation must equal the host pipeline
DeviceFederation(partition_noniid(make_synthetic_dataset(...))) bit for bit.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _bits_equal(a: np.ndarray, b: np.ndarray) -> int:
    """Number of positions whose fp64 bit patterns differ."""
    return int(np.count_nonzero(a.view(np.uint64) != b.view(np.uint64)))


@pytest.mark.parametrize("seed,pre,n", [(0, 0, 0), (0, 0, 1), (1, 0, 7), (12345, 0, 1000),
                                        (7, 3, 1_000_003), (2**63 + 11, 17, 4_000_000),
                                        (99, 0, 20_000_000)])
def test_standard_normal_matches_numpy(seed, pre, n):
    from paper_2305_15668_b200.devicedata import pcg64_standard_normal
    rng = np.random.default_rng(seed)
    if pre:
        rng.integers(0, 10, size=pre)            # start mid-stream, like the dataset's noise draw
    state = rng.bit_generator.state
    got, after = pcg64_standard_normal(state, n)
    want = rng.standard_normal(n)
    torch.cuda.synchronize()
    g = got.cpu().numpy()
    assert g.shape == want.shape
    # every draw decision (fast path / wedge / tail) identical -> same positions, same state; the tail's
    # log1p is glibc's own, so the values are bit-identical too
    assert _bits_equal(g, want) == 0
    assert after["state"]["state"] == rng.bit_generator.state["state"]["state"]
    # the state chains: the next draws agree too
    more, _ = pcg64_standard_normal(after, 1000)
    assert _bits_equal(more.cpu().numpy(), rng.standard_normal(1000)) == 0


def test_standard_normal_rejects_other_generators():
    from paper_2305_15668_b200.devicedata import pcg64_standard_normal
    with pytest.raises(ValueError):
        pcg64_standard_normal(np.random.Generator(np.random.Philox(1)).bit_generator.state, 10)


@pytest.mark.parametrize("F,C,n_total,sizes,alpha", [
    (20, 5, 5000, [300, 0, 517, 1200, 64, 999], 0.5),
    (784, 10, 60_000, [600] * 40 + [1000] * 8, 0.3),
    (50, 62, 40_000, [250] * 100 + [37, 1], 0.1),     # short pools -> the richest-pool path
])
def test_reference_federation_bit_identical(F, C, n_total, sizes, alpha):
    from paper_2305_15668_b200.devicedata import reference_federation
    from paper_2305_15668_b200.experiment import DeviceFederation
    from paper_2305_15668_b200.training import make_synthetic_dataset, partition_noniid
    clients = [(f"c{i:03d}", n) for i, n in enumerate(sizes)]
    train, test = make_synthetic_dataset(F, C, n_total, 21)
    host = DeviceFederation(partition_noniid(train, clients, alpha, 22), test, F, C)
    dev = reference_federation(clients, F, C, n_total, 21, alpha, 22)
    assert dev.offset == host.offset
    assert torch.equal(dev.y, host.y) and torch.equal(dev.y_test, host.y_test)
    assert torch.equal(dev.x, host.x), int((dev.x != host.x).sum())
    assert torch.equal(dev.x_test, host.x_test)
    if host.x_split is not None:
        assert torch.equal(dev.x_split, host.x_split)
