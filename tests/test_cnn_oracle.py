"""CPU checks of the FEMNIST CNN oracle (builder's own oracle; parity unpinned by the reference).

The manual im2col forward/backward of ``oracle.cnn.step`` is pinned to torch
autograd on the same model (F.conv2d / max_pool2d / linear), and the engine's
padded parameter layout round-trips the canonical tensors.
"""

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import cnn as oc


def _autograd_step(p, x, y, lr):
    t = {k: torch.tensor(v, dtype=torch.float64, requires_grad=True) for k, v in p.items()}
    xi = torch.tensor(x, dtype=torch.float64).reshape(-1, 1, 28, 28)
    a = F.max_pool2d(torch.relu(F.conv2d(xi, t["conv1.weight"], t["conv1.bias"], padding=2)), 2)
    a = F.max_pool2d(torch.relu(F.conv2d(a, t["conv2.weight"], t["conv2.bias"], padding=2)), 2)
    h = torch.relu(a.reshape(a.shape[0], -1) @ t["fc1.weight"].T + t["fc1.bias"])
    loss = F.cross_entropy(h @ t["fc2.weight"].T + t["fc2.bias"], torch.tensor(y))
    loss.backward()
    return {k: (v.detach() - lr * v.grad).numpy() for k, v in t.items()}, float(loss)


def test_manual_backward_matches_autograd():
    rng = np.random.default_rng(3)
    C = 10
    p = oc.init_params(C, 7)
    x = rng.normal(size=(16, 784)) * 2.0
    y = rng.integers(0, C, 16)
    want, want_loss = _autograd_step(p, x, y, 0.05)
    t = {k: torch.tensor(v, dtype=torch.float32) for k, v in p.items()}
    loss = oc.step(t, torch.tensor(x, dtype=torch.float32), torch.tensor(y), 0.05, C)
    assert abs(loss - want_loss) < 1e-4 * abs(want_loss)
    for k in p:
        d_got = t[k].numpy() - p[k]
        d_want = want[k] - p[k]
        err = np.abs(d_got - d_want).max() / max(np.abs(d_want).max(), 1e-12)
        assert err < 2e-3, (k, err)


def test_local_train_follows_reference_batch_order():
    """Δ of local_train_cnn == sequential step() over oracle.flmath.batch_plan (fl_core.py:176-189)."""
    from oracle import flmath as fm
    rng = np.random.default_rng(4)
    C = 6
    p = oc.init_params(C, 1)
    x = rng.normal(size=(50, 784))
    y = rng.integers(0, C, 50)
    d, losses = oc.local_train_cnn(p, x, y, 70, 32, 0.1, 9, C)
    assert len(losses) == 3
    t = {k: torch.tensor(v, dtype=torch.float32) for k, v in p.items()}
    xt, yt = torch.tensor(x, dtype=torch.float32), torch.tensor(y)
    for idx in fm.batch_plan(50, 70, 32, 9):
        oc.step(t, xt[idx], yt[idx], 0.1, C)
    for k in p:
        assert np.array_equal(d[k], (t[k] - torch.tensor(p[k], dtype=torch.float32)).numpy())
    empty, _ = oc.local_train_cnn(p, x[:0], y[:0], 70, 32, 0.1, 9, C)
    assert all(not v.any() for v in empty.values())


def test_padded_layout_round_trip():
    from paper_2305_15668_b200.cnn import CnnLayout, init_cnn_params
    for C in (10, 62):
        lay = CnnLayout(C)
        p = init_cnn_params(C, 5)
        ref = oc.init_params(C, 5)
        for k in p:
            assert np.array_equal(p[k], ref[k])
        v = lay.to_padded(p)
        assert v.shape == (lay.P,)
        assert np.count_nonzero(v) == lay.canonical_count
        back = lay.from_padded(v)
        for k in p:
            assert np.array_equal(back[k], p[k]), k
        assert not v[lay.padding_mask()].any()
