"""CPU checks of the MobileNetV2 host layout and oracle (no GPU): the architecture table matches the
oracle's torch state_dict, the padded layout from libfedhc round-trips every canonical tensor, and the
oracle's local_train follows fl_core.local_train's batch plan (one Δ per state tensor, one loss per step)."""

import numpy as np


def test_layout_matches_oracle_and_round_trips():
    from oracle import mobilenet as omb
    from oracle.resnet import state_keys
    from paper_2305_15668_b200.mobilenet import MobilenetLayout, canonical_shapes, init_mobilenet_params
    m = omb.MobileNetV2(10)
    sd = m.state_dict()
    cs = canonical_shapes(10)
    assert [k for k in state_keys(m)] == [n for n, _, _ in cs]
    assert all(tuple(sd[n].shape) == s for n, s, _ in cs)
    assert sum(p.numel() for p in m.parameters()) == 2296922
    lay = MobilenetLayout(10)
    p = init_mobilenet_params(10, 7)
    v = lay.to_padded(p)
    assert v.size == lay.P and lay.P % 64 == 0
    back = lay.from_padded(v)
    assert all(np.array_equal(back[k], p[k]) for k in p)
    assert int((~lay.padding_mask()).sum()) == lay.canonical_count


def test_oracle_local_train_steps():
    from oracle import mobilenet as omb
    from paper_2305_15668_b200.mobilenet import init_mobilenet_params
    rng = np.random.default_rng(0)
    x = rng.standard_normal((24, 3072)).astype(np.float32)
    y = rng.integers(0, 10, 24)
    d, losses = omb.local_train_mobilenet(init_mobilenet_params(10, 1), x, y, 24, 8, 0.05, 5, 10, max_steps=2)
    assert len(losses) == 2 and all(np.isfinite(losses))
    assert np.any(d["linear.weight"]) and np.any(d["bn1.running_mean"])
