"""CIFAR MobileNetV2 client engine (BASELINE config 4; builder-defined model -- no reference CNN exists,
SURVEY §8a a14) vs the torch-CPU oracle (oracle/mobilenet.py): one SGD step of full / ragged / empty
clients, the loss trajectory, graph replay == eager launches, accuracy with running statistics.
Bars as tests/test_resnet_gpu.py (bf16 activations, fp32 accumulation / BN statistics / master weights)."""

import pytest

pytestmark = pytest.mark.gpu


DW_SHAPES = [  # (G, bp, H, C, s)
    (2, 4, 32, 64, 1),
    (1, 4, 32, 192, 2),
    (2, 8, 16, 384, 1),
    (1, 8, 8, 960, 2),
    (3, 16, 4, 960, 1),
]


@pytest.mark.parametrize("G,bp,H,C,s", DW_SHAPES)
def test_depthwise_conv_modes(G, bp, H, C, s):
    """Depthwise 3x3 (pad 1) forward / data gradient / weight gradient + SGD vs torch fp32 on bf16 operands:
    max-abs <= 1e-2 x max|ref| for bf16 outputs, 1e-3 relative for the fp32 weight gradient."""
    import torch
    import torch.nn.functional as F
    from paper_2305_15668_b200 import _abi
    torch.manual_seed(G + bp + H + C + s)
    dev, n, Ho = "cuda", G * bp, H // s
    bf = lambda t: t.to(torch.bfloat16).float()
    x = bf(torch.randn(n, C, H, H))
    w = [bf(torch.randn(C, 1, 3, 3) / 3.0) for _ in range(G)]
    dy = bf(torch.randn(n, C, Ho, Ho))
    sp = torch.cuda.current_stream().cuda_stream
    nhwc = lambda t: t.permute(0, 2, 3, 1).contiguous().to(torch.bfloat16).to(dev)
    xd, dyd = nhwc(x), nhwc(dy)
    wd = torch.stack([t.reshape(C, 9).t() for t in w]).to(torch.bfloat16).to(dev).contiguous()
    y = torch.zeros(n, Ho, Ho, C, dtype=torch.bfloat16, device=dev)
    _abi.check(_abi.lib.fedhc_dw_conv(0, G, bp, H, C, s, xd.data_ptr(), None, wd.data_ptr(), y.data_ptr(), None,
                                      0.0, sp))
    ref = torch.cat([F.conv2d(x[g * bp:(g + 1) * bp], w[g], stride=s, padding=1, groups=C) for g in range(G)])
    torch.cuda.synchronize()
    got = y.float().cpu().permute(0, 3, 1, 2)
    assert (got - ref).abs().max().item() <= 1e-2 * ref.abs().max().item()
    dx = torch.zeros(n, H, H, C, dtype=torch.bfloat16, device=dev)
    _abi.check(_abi.lib.fedhc_dw_conv(1, G, bp, H, C, s, None, dyd.data_ptr(), wd.data_ptr(), dx.data_ptr(), None,
                                      0.0, sp))
    ref = torch.cat([torch.nn.grad.conv2d_input(x[g * bp:(g + 1) * bp].shape, w[g], dy[g * bp:(g + 1) * bp],
                                                stride=s, padding=1, groups=C) for g in range(G)])
    torch.cuda.synchronize()
    got = dx.float().cpu().permute(0, 3, 1, 2)
    assert (got - ref).abs().max().item() <= 1e-2 * ref.abs().max().item()
    master = torch.zeros(G, 9, C, device=dev)
    _abi.check(_abi.lib.fedhc_dw_conv(2, G, bp, H, C, s, xd.data_ptr(), dyd.data_ptr(), None, master.data_ptr(),
                                      None, 1.0, sp))
    torch.cuda.synchronize()
    for g in range(G):
        gw = torch.nn.grad.conv2d_weight(x[g * bp:(g + 1) * bp], w[g].shape, dy[g * bp:(g + 1) * bp], stride=s,
                                         padding=1, groups=C)
        want = -gw.reshape(C, 9).t()
        err = (master[g].cpu() - want).abs().max().item() / want.abs().max().item()
        assert err < 1e-3, (g, err)


class _WL:
    def __init__(self, n, b):
        self.num_samples, self.batch_size = n, b


@pytest.fixture(scope="module")
def msetup():
    import torch
    torch.cuda.set_device(0)
    from paper_2305_15668_b200 import training as tr
    from paper_2305_15668_b200.mobilenet import MobilenetFederation, init_mobilenet_params
    C = 10
    trn, tst = tr.make_synthetic_dataset(3072, C, 400, 23)
    shards = tr.partition_noniid(trn, [("m0", 64), ("m1", 40), ("m2", 0)], 0.5, 4)
    fed = MobilenetFederation(shards, tst, 3072, C).attach_engine(3, 32)
    p = init_mobilenet_params(C, 3)
    params = torch.tensor(fed.layout.to_padded(p), dtype=torch.float64, device="cuda")
    return dict(fed=fed, p=p, params=params, shards=shards, ids=["m0", "m1", "m2"], C=C, tst=tst)


def _rel(a, b):
    import numpy as np
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def test_mobilenet_local_train_vs_oracle(msetup):
    """One SGD step of three clients (m0 full batch of 32, m1 ragged 20 rows + 12 padding images, m2 empty)
    vs the oracle.  First-step gradients of this 52-BN network at initialisation are far more
    ill-conditioned than ResNet-18's: rounding the activations to bf16 alone moves most per-tensor deltas
    by 60-100% (spread = rel(bf16 oracle, fp32 oracle)), and some tensors' exact gradients vanish by
    symmetry (BN bias / running mean behind a BN-linear-BN chain) so only rounding noise is left
    (spread > 2).  Bars: padding entries stay zero; noise-dominated tensors no larger than 3 x the
    oracles' noise;
    running statistics (the forward) within 0.75 x spread + 1e-2 of the bf16-faithful oracle (observed
    0 in the first blocks); every other tensor within about the spread of fp32 and no farther from the
    bf16 oracle than 1.5 x the fp32 distance (coarse, noise-level bounds: e32 <= 1.75 spread + 5e-2, e16 <=
    1.5 spread + 5e-2; summation-order changes move these tensors by that much).  The functional check is the
    next test."""
    import numpy as np
    import torch
    from oracle import flmath as fm
    from oracle import mobilenet as omb
    s = msetup
    fed, lay = s["fed"], s["fed"].layout
    wls = [_WL(32, 32), _WL(20, 32), _WL(32, 32)]
    seeds = [fm.seed_of("train", 1, 0, c) for c in s["ids"]]
    d = fed.train(s["params"], s["ids"], wls, 0.05, seeds)
    torch.cuda.synchronize()
    d = d.cpu().numpy().astype(np.float64)
    p32 = {k: v.astype(np.float32).astype(np.float64) for k, v in s["p"].items()}
    bad = []
    for i, cid in enumerate(s["ids"]):
        assert not d[i][lay.padding_mask()].any()
        got = lay.from_padded(d[i])
        sh = s["shards"][cid]
        args = (p32, sh.features, sh.labels, wls[i].num_samples, wls[i].batch_size, 0.05, seeds[i], s["C"])
        f32, _ = omb.local_train_mobilenet(*args)
        b16, _ = omb.local_train_mobilenet(*args, rounding="bf16")
        for k in f32:
            if not np.any(f32[k]):
                assert np.abs(got[k]).max() <= 1e-5, (cid, k)  # a few fp32 ulps of 1.0 (tiny BN gradients)
                continue
            spread = _rel(b16[k], f32[k])
            e16, e32 = _rel(got[k], b16[k]), _rel(got[k], f32[k])
            if spread > 2:  # vanishing by symmetry: only rounding noise, compare magnitudes
                ok = np.linalg.norm(got[k]) <= 3 * max(np.linalg.norm(b16[k]), np.linalg.norm(f32[k])) + 1e-6
            elif k.endswith(("running_mean", "running_var")):
                ok = e16 <= 0.75 * spread + 1e-2
            else:
                ok = e32 <= 1.75 * spread + 5e-2 and e16 <= 1.5 * spread + 5e-2
            if not ok:
                bad.append((cid, k, round(e16, 4), round(e32, 4), round(spread, 4)))
    assert not bad, bad


def test_mobilenet_update_decreases_loss_like_oracle(msetup):
    """Functional check of the whole backward pass: the engine's one-step delta, applied to the fp32 oracle
    model, lowers the step batch's (train-mode) loss about as much as the fp32 oracle's own delta.  Three
    initialisations at lr 0.01 (first-order regime): the engine reaches 0.94 / 1.07 / 0.94 of the fp32
    decrease (the bf16-faithful oracle 0.99 / 0.94 / 0.90); bars: mean >= 0.85, each >= 0.75.  A gradient
    with a missing or mis-routed term does not get there (a random direction raises the loss)."""
    import numpy as np
    import torch
    import torch.nn.functional as F
    from oracle import flmath as fm
    from oracle import mobilenet as omb
    from oracle.resnet import state_keys
    from paper_2305_15668_b200 import training as tr
    from paper_2305_15668_b200.mobilenet import MobilenetFederation, init_mobilenet_params
    s = msetup
    C, lr = s["C"], 0.01
    trn, tst = tr.make_synthetic_dataset(3072, C, 800, 23)
    shards = tr.partition_noniid(trn, [("t0", 256)], 0.5, 4)
    fed = MobilenetFederation(shards, tst, 3072, C).attach_engine(1, 32)
    seed = fm.seed_of("train", 1, 0, "t0")
    sh = shards["t0"]
    idx = fm.batch_plan(len(sh.labels), 32, 32, seed)[0]
    xt = torch.tensor(sh.features[idx], dtype=torch.float32).reshape(-1, 32, 32, 3).permute(0, 3, 1, 2)
    yt = torch.tensor(sh.labels[idx], dtype=torch.int64)
    ratios = []
    for pseed in (3, 4, 5):
        p = init_mobilenet_params(C, pseed)
        params = torch.tensor(fed.layout.to_padded(p), dtype=torch.float64, device="cuda")
        p32 = {k: v.astype(np.float32).astype(np.float64) for k, v in p.items()}

        def loss(delta):
            m = omb.MobileNetV2(C)
            sd = m.state_dict()
            for k in state_keys(m):
                sd[k].copy_(torch.tensor(p32[k] + (delta[k] if delta is not None else 0.0), dtype=torch.float32))
            m.train()
            with torch.no_grad():
                return float(F.cross_entropy(m(xt), yt))

        got = fed.layout.from_padded(fed.train(params, ["t0"], [_WL(32, 32)], lr, [seed]).cpu().numpy()[0])
        f32, _ = omb.local_train_mobilenet(p32, sh.features, sh.labels, 32, 32, lr, seed, C)
        l0 = loss(None)
        d32 = l0 - loss(f32)
        assert d32 > 0
        ratios.append((l0 - loss(got)) / d32)
    assert np.mean(ratios) >= 0.85 and min(ratios) >= 0.75, ratios


def test_mobilenet_loss_trajectory_matches_oracle(msetup):
    """Mean CE loss of the last local step after 1, 2, 4 and 8 SGD steps within 3% of the fp32 oracle at
    lr 0.01 (observed <= 1.4%, the bf16-faithful oracle's own drift is the same size).  At lr 0.05 this
    network's first steps are chaotic (the loss jumps up at step 4 in every arithmetic) and the bf16
    trajectories drift 5-9% from fp32 by step 6-8, so the trajectory is checked where it is stable."""
    import numpy as np
    import torch
    from oracle import flmath as fm
    from oracle import mobilenet as omb
    from paper_2305_15668_b200 import training as tr
    from paper_2305_15668_b200.mobilenet import MobilenetFederation
    s = msetup
    C, lr = s["C"], 0.01
    trn, tst = tr.make_synthetic_dataset(3072, C, 800, 23)
    shards = tr.partition_noniid(trn, [("t0", 256)], 0.5, 4)
    fed = MobilenetFederation(shards, tst, 3072, C).attach_engine(1, 32)
    params = torch.tensor(fed.layout.to_padded(s["p"]), dtype=torch.float64, device="cuda")
    p32 = {k: v.astype(np.float32).astype(np.float64) for k, v in s["p"].items()}
    seeds = [fm.seed_of("train", 1, 0, "t0")]
    _, l32 = omb.local_train_mobilenet(p32, shards["t0"].features, shards["t0"].labels, 256, 32, lr, seeds[0], C)
    res = []
    for steps in (1, 2, 4, 8):
        fed.train(params, ["t0"], [_WL(32 * steps, 32)], lr, seeds)
        res.append((steps, float(fed.engine.last_loss(1).cpu()[0]), l32[steps - 1]))
    assert all(abs(g - w) <= 0.03 * abs(w) for _, g, w in res), res


def test_mobilenet_graph_equals_eager(msetup):
    import numpy as np
    s = msetup
    from oracle import flmath as fm
    fed = s["fed"]
    wls = [_WL(64, 32), _WL(40, 32), _WL(64, 32)]
    seeds = [fm.seed_of("train", 1, 0, c) for c in s["ids"]]
    a = fed.train(s["params"], s["ids"], wls, 0.05, seeds, use_graph=True).cpu().numpy()
    b = fed.train(s["params"], s["ids"], wls, 0.05, seeds, use_graph=False).cpu().numpy()
    assert np.array_equal(a, b)


def test_mobilenet_eval_matches_oracle(msetup):
    import numpy as np
    import torch
    from oracle import mobilenet as omb
    from oracle.resnet import state_keys
    s = msetup
    m = omb.MobileNetV2(s["C"])
    sd = m.state_dict()
    for k in state_keys(m):
        sd[k].copy_(torch.tensor(s["p"][k], dtype=torch.float32))
    m.eval()
    x = torch.tensor(s["tst"].features, dtype=torch.float32).reshape(-1, 32, 32, 3).permute(0, 3, 1, 2)
    with torch.no_grad():
        logits = m(x).numpy()
    want = int((np.argmax(logits, axis=1) == s["tst"].labels).sum())
    got = s["fed"].correct(s["params"])
    srt = np.sort(logits, axis=1)
    close = int(((srt[:, -1] - srt[:, -2]) < 0.05 * np.abs(srt[:, -1]).max()).sum())
    assert abs(got - want) <= max(2, close), (got, want, close)


def test_mobilenet_heterogeneous_steps_match_solo_runs(msetup):
    """Config 4's non-IID sample counts: clients with 3, 1 and 2 local steps train together (steps after a
    client's last batch run only the clients that still have work, in descending-step order) and each
    client's delta equals -- bit for bit -- the delta of the same client trained alone; its delta row stays
    its own although the engine reorders the descriptors."""
    import numpy as np
    import torch
    from oracle import flmath as fm
    from paper_2305_15668_b200 import training as tr
    from paper_2305_15668_b200.mobilenet import MobilenetFederation
    s = msetup
    C = s["C"]
    trn, tst = tr.make_synthetic_dataset(3072, C, 600, 29)
    ids = ["h0", "h1", "h2"]
    shards = tr.partition_noniid(trn, [("h0", 96), ("h1", 20), ("h2", 60)], 0.5, 4)
    fed = MobilenetFederation(shards, tst, 3072, C).attach_engine(3, 32)
    params = torch.tensor(fed.layout.to_padded(s["p"]), dtype=torch.float64, device="cuda")
    wls = [_WL(96, 32), _WL(20, 32), _WL(60, 32)]
    seeds = [fm.seed_of("train", 2, 0, c) for c in ids]
    n0 = fed.engine.launch_count()
    together = fed.train(params, ids, wls, 0.05, seeds).cpu().numpy()
    assert fed.engine.launch_count() > n0
    for i, cid in enumerate(ids):
        solo = fed.train(params, [cid], [wls[i]], 0.05, [seeds[i]]).cpu().numpy()[0]
        assert np.array_equal(together[i], solo), cid
    loss = fed.engine.last_loss(1).cpu().numpy()
    assert np.isfinite(loss).all()


def test_mobilenet_eval_spans_several_chunks(msetup):
    """Accuracy over a test set far larger than the workspace (one client x batch 8: eleven 8-row chunks, the
    last one ragged) equals a workspace that takes the whole set in one chunk."""
    import torch
    from paper_2305_15668_b200 import training as tr
    from paper_2305_15668_b200.mobilenet import MobilenetFederation
    s = msetup
    trn, tst = tr.make_synthetic_dataset(3072, s["C"], 420, 31)
    shards = tr.partition_noniid(trn, [("e0", 16)], 0.5, 4)
    small = MobilenetFederation(shards, tst, 3072, s["C"]).attach_engine(1, 8)
    big = MobilenetFederation(shards, tst, 3072, s["C"]).attach_engine(3, 32)
    assert small.n_test > 8 and small.n_test % 8 and small.n_test <= 96
    params = torch.tensor(small.layout.to_padded(s["p"]), dtype=torch.float64, device="cuda")
    assert small.correct(params) == big.correct(params)
