"""ResNet client layers on the tcgen05 engine vs torch fp32 on bf16-rounded operands (builder-defined
model: no reference ResNet exists).

NHWC implicit-GEMM convolutions (k = 1 / 3, stride 1 / 2, 4-D TMA boxes with out-of-bounds zero fill as
the padding): forward, data gradient (stride 1; stride 2 runs on the zero-upsampled gradient) and weight
gradient + SGD.  Tolerance: max-abs error <= 1e-2 x max |ref| (bf16 outputs, fp32 accumulation)."""

import pytest

pytestmark = pytest.mark.gpu

SHAPES = [  # (G, bp, H, cin, cout, k, s)
    (2, 4, 32, 64, 64, 3, 1),
    (1, 4, 32, 64, 128, 3, 2),
    (2, 8, 16, 128, 128, 3, 1),
    (1, 8, 16, 128, 256, 1, 2),
    (1, 16, 8, 256, 256, 3, 1),
    (2, 32, 4, 512, 512, 3, 1),
    (1, 32, 8, 256, 512, 3, 2),
]


def _w_layout(w):
    """torch [cout, cin, k, k] -> engine [k*k*cin][cout] (tap-major)."""
    co, ci, k, _ = w.shape
    return w.permute(2, 3, 1, 0).reshape(k * k * ci, co)


@pytest.mark.parametrize("G,bp,H,cin,cout,k,s", SHAPES)
def test_nhwc_conv_modes(G, bp, H, cin, cout, k, s):
    import torch
    import torch.nn.functional as F
    from paper_2305_15668_b200 import _abi
    torch.manual_seed(G * 100 + H + cin + k + s)
    dev = "cuda"
    n, Ho = G * bp, H // s
    bf = lambda t: t.to(torch.bfloat16).float()
    x = bf(torch.randn(n, cin, H, H))
    w = [bf(torch.randn(cout, cin, k, k) * (1.0 / (k * k * cin) ** 0.5)) for _ in range(G)]
    dy = bf(torch.randn(n, cout, Ho, Ho))
    sp = torch.cuda.current_stream().cuda_stream
    xd = x.permute(0, 2, 3, 1).contiguous().to(torch.bfloat16).to(dev)
    wd = torch.stack([_w_layout(t) for t in w]).to(torch.bfloat16).to(dev).contiguous()
    pad = k // 2
    # forward
    y = torch.zeros(n, Ho, Ho, cout, dtype=torch.bfloat16, device=dev)
    _abi.check(_abi.lib.fedhc_nhwc_conv(4, G, bp, H, H, cin, cout, k, s, xd.data_ptr(), None, wd.data_ptr(),
                                        y.data_ptr(), None, 0.0, sp))
    ref = torch.cat([F.conv2d(x[g * bp:(g + 1) * bp], w[g], stride=s, padding=pad) for g in range(G)])
    torch.cuda.synchronize()
    got = y.float().cpu().permute(0, 3, 1, 2)
    assert (got - ref).abs().max().item() <= 1e-2 * ref.abs().max().item()
    # data gradient: stride 1 directly; stride 2 through the zero-upsampled output gradient
    u = torch.zeros(n, cout, H, H)
    u[:, :, ::s, ::s] = dy
    ud = u.permute(0, 2, 3, 1).contiguous().to(torch.bfloat16).to(dev)
    dx = torch.zeros(n, H, H, cin, dtype=torch.bfloat16, device=dev)
    _abi.check(_abi.lib.fedhc_nhwc_conv(5, G, bp, H, H, cin, cout, k, 1, None, ud.data_ptr(), wd.data_ptr(),
                                        dx.data_ptr(), None, 0.0, sp))
    ref = torch.cat([torch.nn.grad.conv2d_input(x[g * bp:(g + 1) * bp].shape, w[g], dy[g * bp:(g + 1) * bp],
                                                stride=s, padding=pad) for g in range(G)])
    torch.cuda.synchronize()
    got = dx.float().cpu().permute(0, 3, 1, 2)
    assert (got - ref).abs().max().item() <= 1e-2 * ref.abs().max().item()
    # weight gradient + SGD (lr = 1, zero master): master = -grad
    dyd = dy.permute(0, 2, 3, 1).contiguous().to(torch.bfloat16).to(dev)
    master = torch.zeros(G, k * k * cin, cout, device=dev)
    _abi.check(_abi.lib.fedhc_nhwc_conv(6, G, bp, H, H, cin, cout, k, s, xd.data_ptr(), dyd.data_ptr(), None,
                                        master.data_ptr(), None, 1.0, sp))
    torch.cuda.synchronize()
    for g in range(G):
        gw = torch.nn.grad.conv2d_weight(x[g * bp:(g + 1) * bp], w[g].shape, dy[g * bp:(g + 1) * bp], stride=s,
                                         padding=pad)
        want = -_w_layout(gw)
        err = (master[g].cpu() - want).abs().max().item() / want.abs().max().item()
        assert err < 1e-3, (g, err)


# ---- ResNet-18 client engine vs the fp32 torch-CPU oracle (oracle/resnet.py) -----------------------
class _WL:
    def __init__(self, n, b):
        self.num_samples, self.batch_size = n, b


@pytest.fixture(scope="module")
def rsetup():
    import torch
    torch.cuda.set_device(0)
    from paper_2305_15668_b200 import training as tr
    from paper_2305_15668_b200.resnet import ResnetFederation, init_resnet_params
    C = 10
    trn, tst = tr.make_synthetic_dataset(3072, C, 400, 21)
    shards = tr.partition_noniid(trn, [("r0", 64), ("r1", 40), ("r2", 0)], 0.5, 4)
    fed = ResnetFederation(shards, tst, 3072, C).attach_engine(3, 32)
    p = init_resnet_params(C, 2)
    params = torch.tensor(fed.layout.to_padded(p), dtype=torch.float64, device="cuda")
    return dict(fed=fed, p=p, params=params, shards=shards, ids=["r0", "r1", "r2"], C=C, tst=tst)


def _rel(a, b):
    import numpy as np
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def test_resnet_local_train_vs_oracle(rsetup):
    """One SGD step of three clients (r0: a full batch of 32; r1: a ragged batch of 20 rows -- the 12
    padding images must not touch the batch statistics or the gradients; r2: empty shard) vs the
    torch-CPU oracle.

    First-step gradients of a batch-norm network at initialisation are ill-conditioned: rounding the
    activations to bf16 alone moves the per-tensor deltas by up to ~30% (spread = rel(bf16 oracle, fp32
    oracle)) while the forward and the loss trajectory agree closely (next test).  Bars: running
    statistics (the forward) within 1e-2 of the bf16-faithful oracle; classifier deltas within 2e-2 of
    fp32; every other tensor within 1.5 x spread + 2e-2 of fp32 and cosine(engine, fp32) within 0.05 of
    cosine(bf16 oracle, fp32) -- a missing or mis-routed gradient term fails these by a wide margin."""
    import numpy as np
    import torch
    from oracle import flmath as fm
    from oracle import resnet as orn
    s = rsetup
    fed, lay = s["fed"], s["fed"].layout
    wls = [_WL(32, 32), _WL(20, 32), _WL(32, 32)]
    seeds = [fm.seed_of("train", 1, 0, c) for c in s["ids"]]
    d = fed.train(s["params"], s["ids"], wls, 0.05, seeds)
    torch.cuda.synchronize()
    d = d.cpu().numpy().astype(np.float64)
    p32 = {k: v.astype(np.float32).astype(np.float64) for k, v in s["p"].items()}
    cosf = lambda a, b: float(np.dot(a.ravel(), b.ravel()) / max(np.linalg.norm(a) * np.linalg.norm(b), 1e-30))
    for i, cid in enumerate(s["ids"]):
        assert not d[i][lay.padding_mask()].any()
        got = lay.from_padded(d[i])
        sh = s["shards"][cid]
        args = (p32, sh.features, sh.labels, wls[i].num_samples, wls[i].batch_size, 0.05, seeds[i], s["C"])
        f32, _ = orn.local_train_resnet(*args)
        b16, _ = orn.local_train_resnet(*args, rounding="bf16")
        for k in f32:
            if not np.any(f32[k]):
                assert np.abs(got[k]).max() <= 1e-6, (cid, k)
                continue
            spread = _rel(b16[k], f32[k])
            e16, e32 = _rel(got[k], b16[k]), _rel(got[k], f32[k])
            if k.endswith(("running_mean", "running_var")):
                assert e16 <= 1e-2, (cid, k, e16)
            elif k.startswith("linear"):
                assert e32 <= 2e-2, (cid, k, e32)
            else:
                assert e32 <= 1.5 * spread + 2e-2, (cid, k, e32, spread)
                assert cosf(got[k], f32[k]) >= min(0.9, cosf(b16[k], f32[k]) - 0.05), (cid, k)


def test_resnet_loss_trajectory_matches_oracle(rsetup):
    """The training trajectory: the engine's mean CE loss of the last local step after 1, 2 and 4 SGD steps
    agrees with the fp32 oracle's within 3% (observed < 1.2%)."""
    import numpy as np
    import torch
    from oracle import flmath as fm
    from oracle import resnet as orn
    from paper_2305_15668_b200 import training as tr
    from paper_2305_15668_b200.resnet import ResnetFederation
    s = rsetup
    C = s["C"]
    trn, tst = tr.make_synthetic_dataset(3072, C, 800, 21)
    shards = tr.partition_noniid(trn, [("t0", 256)], 0.5, 4)
    fed = ResnetFederation(shards, tst, 3072, C).attach_engine(1, 32)
    params = torch.tensor(fed.layout.to_padded(s["p"]), dtype=torch.float64, device="cuda")
    p32 = {k: v.astype(np.float32).astype(np.float64) for k, v in s["p"].items()}
    seeds = [fm.seed_of("train", 1, 0, "t0")]
    for steps in (1, 2, 4):
        fed.train(params, ["t0"], [_WL(32 * steps, 32)], 0.05, seeds)
        got = float(fed.engine.last_loss(1).cpu()[0])
        _, l32 = orn.local_train_resnet(p32, shards["t0"].features, shards["t0"].labels, 32 * steps, 32, 0.05,
                                        seeds[0], C)
        assert abs(got - l32[-1]) <= 0.03 * abs(l32[-1]), (steps, got, l32[-1])


def test_resnet_graph_equals_eager(rsetup):
    import numpy as np
    import torch
    from oracle import flmath as fm
    s = rsetup
    fed = s["fed"]
    wls = [_WL(64, 32), _WL(40, 32), _WL(64, 32)]
    seeds = [fm.seed_of("train", 1, 0, c) for c in s["ids"]]
    a = fed.train(s["params"], s["ids"], wls, 0.05, seeds, use_graph=True).cpu().numpy()
    b = fed.train(s["params"], s["ids"], wls, 0.05, seeds, use_graph=False).cpu().numpy()
    assert np.array_equal(a, b)


def test_resnet_eval_matches_oracle(rsetup):
    import numpy as np
    import torch
    from oracle import resnet as orn
    s = rsetup
    m = orn.ResNet18(s["C"])
    sd = m.state_dict()
    for k in orn.state_keys(m):
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
