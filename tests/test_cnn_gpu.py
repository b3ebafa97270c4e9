"""FEMNIST CNN engine (tcgen05 grouped GEMMs) vs the torch-CPU oracle.

Tolerances (bf16 tensor-core operands, fp32 accumulation and fp32 master
weights; the oracle is the builder's own -- parity unpinned by the reference),
per tensor, rel = ||Δ_gpu − Δ_oracle|| / ||Δ_oracle||:
  * vs the bf16-faithful oracle (same rounding points):
    rel <= max(1e-2, 0.75 * spread), spread = rel(bf16 oracle, fp32 oracle),
    and closer to it than to the fp32 oracle -- the engine must sit closer to
    its own rounding model than bf16 sits to fp32 (SGD amplifies any rounding
    difference step by step; after 1 step rel is ~1e-3);
  * vs the plain fp32 oracle: rel <= max(6e-2, 2 * spread);
  * layout padding of every delta exactly 0; graph replay == eager launches
    bit for bit; repeated runs bit-identical.
"""

import numpy as np
import pytest

from oracle import cnn as ocnn
from oracle import flmath as fm

pytestmark = pytest.mark.gpu

LR = 0.01


def _rel(got, want):
    return float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-30))


class WL:
    def __init__(self, n, b):
        self.num_samples, self.batch_size = n, b


@pytest.fixture(scope="module")
def setup():
    import torch
    torch.cuda.set_device(0)
    from paper_2305_15668_b200 import training as tr
    from paper_2305_15668_b200.cnn import CnnFederation, init_cnn_params
    C = 10
    trn, tst = tr.make_synthetic_dataset(784, C, 1600, 11)
    ids = ["c0", "c1", "c2", "c3"]
    shards = tr.partition_noniid(trn, [("c0", 256), ("c1", 300), ("c2", 0), ("c3", 130)], 0.5, 3)
    fed = CnnFederation(shards, tst, 784, C).attach_engine(4, 64)
    p = init_cnn_params(C, 1)
    params = torch.tensor(fed.layout.to_padded(p), dtype=torch.float64, device="cuda")
    return dict(fed=fed, p=p, params=params, shards=shards, ids=ids, C=C, tst=tst)


def _run(s, wls, steps=None, use_graph=True, lr=LR):
    import torch
    fed = s["fed"]
    seeds = [fm.seed_of("train", 1, 0, c) for c in s["ids"]]
    if steps is not None:   # truncate every client's local loop to `steps` batches
        wls = [WL(min(w.num_samples, steps * w.batch_size), w.batch_size) for w in wls]
    d = fed.train(s["params"], s["ids"], wls, lr, seeds, use_graph=use_graph)
    torch.cuda.synchronize()
    return d.cpu().numpy().astype(np.float64), seeds, wls


def _oracle(s, cid, wl, seed, rounding, lr=LR):
    sh = s["shards"][cid]
    p32 = {k: v.astype(np.float32).astype(np.float64) for k, v in s["p"].items()}
    return ocnn.local_train_cnn(p32, sh.features, sh.labels, wl.num_samples, wl.batch_size, lr, seed, s["C"],
                                rounding=rounding)[0]


@pytest.mark.parametrize("steps", [1, 3, 6])
def test_cnn_local_train_vs_oracles(setup, steps):
    """Deltas vs both oracles; ragged (c1: 300 = 4*64 + 44), empty (c2) and shorter (c3) clients."""
    s = setup
    wls = [WL(256, 64), WL(300, 64), WL(64, 64), WL(200, 64)]
    d, seeds, wls = _run(s, wls, steps)
    lay = s["fed"].layout
    for i, cid in enumerate(s["ids"]):
        assert not d[i][lay.padding_mask()].any()
        got = lay.from_padded(d[i])
        b16 = _oracle(s, cid, wls[i], seeds[i], "bf16")
        f32 = _oracle(s, cid, wls[i], seeds[i], None)
        for k in b16:
            if not np.any(b16[k]):
                assert not np.any(got[k]), (cid, k)
                continue
            spread = _rel(b16[k], f32[k])          # bf16's own deviation from fp32 on this trajectory
            e16, e32 = _rel(got[k], b16[k]), _rel(got[k], f32[k])
            assert e16 <= max(1e-2, 0.75 * spread), (cid, k, e16, spread)
            assert e16 <= max(1e-2, e32), (cid, k, e16, e32)
            assert e32 <= max(6e-2, 2.0 * spread), (cid, k, e32, spread)


def test_cnn_graph_equals_eager_and_deterministic(setup):
    s = setup
    wls = [WL(256, 64), WL(300, 64), WL(64, 64), WL(200, 64)]
    a, _, _ = _run(s, wls, use_graph=True)
    b, _, _ = _run(s, wls, use_graph=False)
    c, _, _ = _run(s, wls, use_graph=True)
    assert np.array_equal(a, b) and np.array_equal(a, c)


def test_cnn_eval_matches_oracle_predictions(setup):
    s = setup
    fed, tst = s["fed"], s["tst"]
    logits = ocnn.forward_logits(s["p"], tst.features)
    want = int((np.argmax(logits, axis=1) == tst.labels).sum())
    got = fed.correct(s["params"])
    # bf16 operands: only near-tied logits may flip
    margin = np.sort(logits, axis=1)
    close = int(((margin[:, -1] - margin[:, -2]) < 0.05 * np.abs(margin[:, -1]).max()).sum())
    assert abs(got - want) <= max(2, close), (got, want, close)


# ---- conv2 implicit GEMM (TMA 4-D boxes, OOB zero padding) vs torch fp32 on bf16 operands ----------
def _pairs_layout(w):
    """torch conv2 weight [64 co, 32 ci, 5, 5] -> engine [16 pairs][2][32 ci][64 co] (kw = 5, pair 15 zero)."""
    import torch
    t = torch.zeros(5, 6, 32, 64)
    t[:, :5] = w.permute(2, 3, 1, 0)
    out = torch.zeros(16, 2, 32, 64)
    out[:15] = t.reshape(15, 2, 32, 64)
    return out.reshape(1024, 64)


def _p1x(p1):
    """p1 NHWC [n,14,14,32] -> channel pairs [n,14,15,64]: column xx = p1(y,xx-1) | p1(y,xx), zero outside."""
    import torch
    n = p1.shape[0]
    pad = torch.zeros(n, 14, 16, 32)
    pad[:, :, 1:15] = p1
    return torch.cat([pad[:, :, 0:15], pad[:, :, 1:16]], dim=3)


@pytest.mark.parametrize("G,bp", [(1, 1), (3, 2)])
def test_conv2_implicit_gemm_modes(G, bp):
    import torch
    import torch.nn.functional as Fn
    from paper_2305_15668_b200 import _abi
    torch.manual_seed(G * 10 + bp)
    dev = "cuda"
    n = G * bp
    bf = lambda t: t.to(torch.bfloat16).float()
    p1 = bf(torch.randn(n, 14, 14, 32))
    w = [bf(torch.randn(64, 32, 5, 5) * 0.05) for _ in range(G)]
    bias = torch.randn(G, 64) * 0.1
    da2 = bf(torch.randn(n, 14, 14, 64))
    wl = torch.stack([_pairs_layout(x) for x in w]).to(torch.bfloat16).to(dev)
    p1x = _p1x(p1).to(torch.bfloat16).to(dev).contiguous()
    sp = torch.cuda.current_stream().cuda_stream
    # forward
    out = torch.zeros(n, 14, 14, 64, dtype=torch.bfloat16, device=dev)
    b_dev = bias.to(dev).contiguous()
    _abi.check(_abi.lib.fedhc_cnn_conv2(1, G, bp, p1x.data_ptr(), None, wl.data_ptr(), b_dev.data_ptr(),
                                        out.data_ptr(), 0.0, sp))
    ref = torch.cat([Fn.conv2d(p1[g * bp:(g + 1) * bp].permute(0, 3, 1, 2), w[g], bias[g], padding=2)
                     for g in range(G)]).relu().permute(0, 2, 3, 1)
    torch.cuda.synchronize()
    err = (out.float().cpu() - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-2, err
    # data gradient: dL/dp1 = conv_transpose(dL/da2)
    dp1 = torch.zeros(n, 14, 14, 32, dtype=torch.bfloat16, device=dev)
    da2_dev = da2.to(torch.bfloat16).to(dev).contiguous()
    _abi.check(_abi.lib.fedhc_cnn_conv2(2, G, bp, da2_dev.data_ptr(), None, wl.data_ptr(), None, dp1.data_ptr(),
                                        0.0, sp))
    ref = torch.cat([Fn.conv_transpose2d(da2[g * bp:(g + 1) * bp].permute(0, 3, 1, 2), w[g], padding=2)
                     for g in range(G)]).permute(0, 2, 3, 1)
    torch.cuda.synchronize()
    err = (dp1.float().cpu() - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-2, err
    # weight gradient + SGD on an fp32 master (zero start): master = -lr * grad
    master = torch.zeros(G, 1024, 64, device=dev)
    _abi.check(_abi.lib.fedhc_cnn_conv2(3, G, bp, p1x.data_ptr(), da2_dev.data_ptr(), None, None, master.data_ptr(),
                                        1.0, sp))
    torch.cuda.synchronize()
    for g in range(G):
        x = p1[g * bp:(g + 1) * bp].permute(0, 3, 1, 2)
        gy = da2[g * bp:(g + 1) * bp].permute(0, 3, 1, 2)
        gw = torch.nn.grad.conv2d_weight(x, (64, 32, 5, 5), gy, padding=2)
        want = -_pairs_layout(gw)
        got = master[g].cpu()
        pad = _pairs_layout(torch.ones(64, 32, 5, 5)) == 0          # kw = 5 rows, pair 15
        real = ~pad
        err = (got[real] - want[real]).abs().max().item() / want.abs().max().item()
        assert err < 1e-3, (g, err)
        assert not got.reshape(16, 2, 32, 64)[15].any()           # padding pair: fully out-of-bounds boxes
