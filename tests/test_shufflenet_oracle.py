"""CPU checks of the ShuffleNetV2 host layout and oracle (no GPU): architecture table == the oracle's torch
state_dict, the split-form padded layout from libfedhc round-trips every canonical tensor, the channel
shuffle is the 2-group transpose, and the oracle's local_train follows fl_core.local_train's batch plan."""

import numpy as np


def test_layout_matches_oracle_and_round_trips():
    from oracle import shufflenet as osn
    from oracle.resnet import state_keys
    from paper_2305_15668_b200.shufflenet import ShufflenetLayout, canonical_shapes, init_shufflenet_params
    m = osn.ShuffleNetV2(10)
    sd = m.state_dict()
    cs = canonical_shapes(10)
    assert [k for k in state_keys(m)] == [c[0] for c in cs]
    assert all(tuple(sd[c[0]].shape) == c[1] for c in cs)
    assert sum(p.numel() for p in m.parameters()) == 1263854
    lay = ShufflenetLayout(10)
    p = init_shufflenet_params(10, 7)
    back = lay.from_padded(lay.to_padded(p))
    assert all(np.array_equal(back[k], p[k]) for k in p)
    assert int((~lay.padding_mask()).sum()) == lay.canonical_count


def test_channel_shuffle_is_group_transpose():
    import torch
    from oracle.shufflenet import shuffle
    x = torch.arange(2 * 6).float().reshape(1, 12, 1, 1)
    assert shuffle(x).flatten().tolist() == [0, 6, 1, 7, 2, 8, 3, 9, 4, 10, 5, 11]


def test_oracle_local_train_steps():
    from oracle import shufflenet as osn
    from paper_2305_15668_b200.shufflenet import init_shufflenet_params
    rng = np.random.default_rng(0)
    x = rng.standard_normal((24, 3072)).astype(np.float32)
    y = rng.integers(0, 10, 24)
    d, losses = osn.local_train_shufflenet(init_shufflenet_params(10, 1), x, y, 24, 8, 0.05, 5, 10, max_steps=2)
    assert len(losses) == 2 and all(np.isfinite(losses))
    assert np.any(d["linear.weight"]) and np.any(d["bn1.running_mean"])
