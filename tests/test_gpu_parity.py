"""GPU parity: the CUDA path through the C-ABI vs the CPU oracle and the
reference goldens.

Tolerances (north_star): aggregated weights max-abs <= 1e-4 x max|ref|
after a round (fp32 storage, bf16x3 products; observed ~1e-6); FedAvg and
loss_and_grad are fp64 (FedAvg bit-exact for fp64 deltas); accuracy within
2 test rows of the oracle (argmax near-ties can flip under fp32 logits).
"""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import flmath as fm
from oracle import orchestration as oc

pytestmark = pytest.mark.gpu

REL = 1e-4


def rel_err(got, want):
    scale = max(np.max(np.abs(want)), 1e-30)
    return float(np.max(np.abs(np.asarray(got) - np.asarray(want))) / scale)


@pytest.fixture(scope="module")
def fh():
    import torch
    torch.cuda.set_device(0)
    import paper_2305_15668_b200 as mod
    return mod


@pytest.fixture(scope="module")
def tr(fh):
    from paper_2305_15668_b200 import training
    return training


FL = np.load(os.path.join(GOLDEN, "flcore.npz"))


@pytest.mark.parametrize("i", range(6))
def test_local_train_golden_cases(tr, i):
    F, C, n, ns, b, lr = FL["lt_cases"][i]
    F, C, n, ns, b = int(F), int(C), int(n), int(ns), int(b)
    sd = str(FL["lt_seeds"][i])
    seed = int(sd) if sd.lstrip("-").isdigit() else sd
    shard = tr.DatasetShard("a", FL[f"lt{i}_x"], FL[f"lt{i}_y"])
    from paper_2305_15668_b200.spec import WorkloadSpec
    d = tr.local_train(FL[f"lt{i}_p"], shard, WorkloadSpec(ns, b), float(lr), C, seed=seed)
    want = FL[f"lt{i}_d"]
    if n == 0:
        assert np.all(d == 0)
    else:
        assert rel_err(d, want) <= REL


@pytest.mark.parametrize("F,C,n,ns,b", [
    (784, 10, 640, 640, 64),     # FEMNIST-shaped, fast path (NT=2)
    (784, 10, 300, 1000, 64),    # reshuffles + ragged batch before each reshuffle
    (784, 10, 100, 100, 32),     # ragged last batch (100 = 3*32 + 4)
    (784, 32, 256, 256, 64),     # NT=4 fast path
    (784, 3, 128, 128, 64),      # NT=1
    (784, 8, 200, 200, 64),      # split-row trainer, classes 0-7 only
    (784, 12, 200, 300, 64),     # split-row trainer, packed [Wh | Wm] tile of classes 8..11, reshuffle
    (784, 16, 256, 256, 64),     # split-row trainer, two class tiles
    (784, 62, 256, 256, 64),     # FEMNIST 62 classes (2-CTA tcgen05 trainer, master in TMEM, SW32 tail)
    (784, 62, 100, 300, 64),     # 62 classes, ragged + reshuffle
    (744, 50, 150, 300, 64),     # 2-CTA trainer: partial SW128 last chunk (40 features)
    (200, 40, 120, 240, 48),     # 2-CTA trainer: lone chunk tile + 8-feature SW32 tail, B not a multiple of 16
    (128, 33, 64, 64, 64),       # 2-CTA trainer: one chunk per CTA
    (72, 64, 90, 90, 30),        # 2-CTA trainer: CTA 1 holds only the tail
    (784, 20, 128, 128, 64),     # 2-CTA cluster, partial second class slice
    (392, 40, 96, 96, 32),       # cluster path, F not filling all warps
    (64, 10, 200, 300, 50),      # small F, B not a multiple of 16
    (20, 7, 90, 90, 1),          # batch of one row
    (6, 4, 33, 66, 16),          # F % 4 != 0 -> generic path
    (3072, 10, 200, 640, 64),    # CIFAR-shaped reference model: tcgen05 trainer, 8-CTA clusters
    (1000, 40, 150, 300, 32),    # tcgen05 trainer, odd chunk count per CTA, ragged + reshuffle
    (784, 64, 128, 256, 64),     # tcgen05 trainer at the full 64-class tile
    (2, 10, 6400, 6400, 6400),   # the reference's default F = 2, one 6400-row batch: generic, row-tiled
    (16, 100, 300, 300, 64),     # more than 64 classes: generic
])
def test_local_train_vs_oracle(tr, F, C, n, ns, b):
    from paper_2305_15668_b200.spec import WorkloadSpec
    trn, _ = fm.synthetic(F, C, n * 2 + 10, seed=F + C + n)
    shard = fm.Shard("a", trn.features[:n], trn.labels[:n])
    params = np.random.default_rng(1).standard_normal(F * C + C) * 0.05
    want = fm.local_sgd(params, shard, ns, b, 0.1, C, seed=17)
    got = tr.local_train(params, tr.DatasetShard("a", shard.features, shard.labels), WorkloadSpec(ns, b), 0.1, C,
                         seed=17)
    assert rel_err(got, want) <= REL, rel_err(got, want)


def test_local_train_does_not_mutate(tr):
    from paper_2305_15668_b200.spec import WorkloadSpec
    trn, _ = fm.synthetic(8, 4, 200, seed=9)
    params = np.zeros(36)
    tr.local_train(params, tr.DatasetShard("a", trn.features[:100], trn.labels[:100]), WorkloadSpec(100, 32), 0.1, 4)
    assert np.array_equal(params, np.zeros(36))


def test_local_train_deterministic(tr):
    from paper_2305_15668_b200.spec import WorkloadSpec
    trn, _ = fm.synthetic(784, 10, 900, seed=3)
    sh = tr.DatasetShard("a", trn.features[:700], trn.labels[:700])
    a = tr.local_train(np.zeros(7850), sh, WorkloadSpec(700, 64), 0.1, 10, seed=5)
    b = tr.local_train(np.zeros(7850), sh, WorkloadSpec(700, 64), 0.1, 10, seed=5)
    assert np.array_equal(a, b)


def test_fedavg_bit_exact(tr):
    out = tr.fedavg(list(FL["fa_deltas"]), list(FL["fa_w"]), FL["fa_base"])
    assert np.array_equal(out, FL["fa_out"])
    base = np.array([1.0, 1.0])
    ds = [np.array([2.0, 4.0]), np.array([4.0, 6.0])]
    assert np.array_equal(tr.fedavg(ds, [1.0, 1.0], base), [4.0, 6.0])
    assert np.array_equal(tr.fedavg(ds, [3.0, 1.0], base), [3.5, 5.5])
    rng = np.random.default_rng(4)
    for n, k in [(1, 1), (3, 2), (4097, 9), (100_003, 37)]:
        base = rng.standard_normal(n)
        ds = [rng.standard_normal(n) for _ in range(k)]
        ws = list(rng.uniform(0.1, 5.0, size=k))
        assert np.array_equal(tr.fedavg(ds, ws, base), fm.weighted_average(ds, ws, base))


def test_fedavg_short_vectors_pointer_rows(tr):
    """The shared-memory tile kernel (short vectors): fp32 pointer-table rows as the round loop passes them,
    16-byte aligned and misaligned, K above one staged tile, ragged tails; bit-exact vs torch fp64 in list order."""
    import torch
    from paper_2305_15668_b200 import _abi
    g = torch.Generator(device="cuda").manual_seed(3)
    for n, k, shift in [(7850, 100, 0), (7850, 100, 1), (130, 300, 0), (1, 3, 0), (129, 129, 3)]:
        ld = (n + 3) // 4 * 4 + 4
        store = torch.randn(k, ld, device="cuda", generator=g, dtype=torch.float32)
        rows = store[:, shift:shift + n]
        table = torch.tensor([r.data_ptr() for r in rows], dtype=torch.int64, device="cuda")
        coef = torch.rand(k, device="cuda", generator=g, dtype=torch.float64)
        base = torch.randn(n, device="cuda", generator=g, dtype=torch.float64)
        out = torch.empty_like(base)
        _abi.check(_abi.lib.fedhc_fedavg(table.data_ptr(), None, 0, _abi.F32, coef.data_ptr(), k, base.data_ptr(),
                                         out.data_ptr(), n, torch.cuda.current_stream().cuda_stream))
        ref = base.clone()
        for i in range(k):
            ref += coef[i].item() * rows[i].double()
        assert torch.equal(out, ref), (n, k, shift)


def test_fedavg_errors(tr):
    from paper_2305_15668_b200.errors import AggregationError
    for ds, ws in [([], []), ([np.zeros(2)], [1.0, 2.0]), ([np.zeros(3)], [1.0]), ([np.zeros(2)], [0.0]),
                   ([np.zeros(2)], [-1.0])]:
        with pytest.raises(AggregationError):
            tr.fedavg(ds, ws, np.zeros(2))


def test_fedavg_full_size_vs_torch(tr):
    """Config-5 scale (P = 25M, K = 8, fp32 deltas): bit-exact vs the same sequence in torch fp64."""
    import torch
    P, K = 25_000_000, 8
    g = torch.Generator(device="cuda").manual_seed(0)
    deltas = torch.randn(K, P, device="cuda", generator=g, dtype=torch.float32) * 1e-3
    base = torch.randn(P, device="cuda", generator=g, dtype=torch.float64)
    w = [float(v) for v in torch.randint(1, 1024, (K,), generator=torch.Generator().manual_seed(0))]
    total = float(sum(w))
    coef = torch.tensor([x / total for x in w], dtype=torch.float64, device="cuda")
    out = torch.empty_like(base)
    tr.fedavg_device(deltas, coef, base, out)
    ref = base.clone()
    for k in range(K):
        ref += coef[k].item() * deltas[k].double()
    assert torch.equal(out, ref)
    # properties: single delta with any weight -> base + delta exactly; zero deltas -> base
    tr.fedavg_device(deltas[:1], torch.tensor([1.0], dtype=torch.float64, device="cuda"), base, out)
    assert torch.equal(out, base + deltas[0].double())


@pytest.mark.parametrize("P,K", [(1_000_003, 37), (250_004, 600), (4097, 1000), (2_000_000, 33)])
def test_fedavg_tma_streamed_vs_torch(tr, P, K):
    """The TMA-fed persistent FedAvg (packed rows, P <= 4M or K >= 500; ragged last segment, many row groups,
    fewer rows than one stage): bit-exact vs the same list-order sequence in torch fp64."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(P + K)
    ld = (P + 3) // 4 * 4
    deltas = (torch.randn(K, ld, device="cuda", generator=g, dtype=torch.float32) * 1e-3)[:, :P]
    base = torch.randn(P, device="cuda", generator=g, dtype=torch.float64)
    w = torch.rand(K, generator=torch.Generator().manual_seed(K), dtype=torch.float64) + 0.1
    coef = (w / w.sum()).cuda()
    out = torch.empty_like(base)
    tr.fedavg_device(deltas, coef, base, out)
    ref = base.clone()
    for k in range(K):
        ref += coef[k].item() * deltas[k].double()
    assert torch.equal(out, ref)
    tr.fedavg_device(deltas, coef, None, out)  # partial sums (multi-GPU path): no base
    ref = torch.zeros_like(base)
    for k in range(K):
        ref += coef[k].item() * deltas[k].double()
    assert torch.equal(out, ref)


def test_accuracy_vs_oracle(tr):
    d = fm.Data(FL["acc_x"], FL["acc_y"], 6)
    assert tr.evaluate_accuracy(FL["acc_p"], tr.Dataset(d.features, d.labels, 6)) == fm.accuracy(FL["acc_p"], d)
    trn, tst = fm.synthetic(784, 62, 5000, seed=2)
    p = np.random.default_rng(0).standard_normal(784 * 62 + 62) * 0.01
    got = tr.evaluate_accuracy(p, tr.Dataset(tst.features, tst.labels, 62))
    assert abs(got - fm.accuracy(p, tst)) <= 2 / len(tst.labels)
    assert tr.evaluate_accuracy(p, tr.Dataset(np.zeros((0, 784)), np.zeros(0, int), 62)) == 0.0
    # a model too large for shared memory (3072 x 100 fp32 = 1.2 MB): W read from global memory
    trn, tst = fm.synthetic(3072, 100, 3000, seed=4)
    p = np.random.default_rng(1).standard_normal(3072 * 100 + 100) * 0.01
    got = tr.evaluate_accuracy(p, tr.Dataset(tst.features, tst.labels, 100))
    assert abs(got - fm.accuracy(p, tst)) <= 2 / len(tst.labels)


def test_accuracy_cta_cap_invariant():
    """fedhc_eval_ctas (the round loop's accuracy on the SMs training leaves idle) counts exactly what
    fedhc_eval counts, for any CTA cap, on ragged row counts."""
    import torch
    from paper_2305_15668_b200 import _abi
    g = torch.Generator(device="cuda").manual_seed(7)
    for n, F, C in [(16000, 784, 10), (1001, 784, 62), (33, 60, 3)]:
        x = torch.randn(n, F, device="cuda", generator=g)
        y = torch.randint(0, C, (n,), device="cuda", generator=g, dtype=torch.int32)
        p = torch.randn(F * C + C, device="cuda", generator=g, dtype=torch.float64) * 0.05
        st = torch.cuda.current_stream().cuda_stream
        ref = torch.zeros(1, dtype=torch.int64, device="cuda")
        _abi.check(_abi.lib.fedhc_eval(x.data_ptr(), y.data_ptr(), n, F, C, p.data_ptr(), ref.data_ptr(), st))
        expect = int(((x.double() @ p[:F * C].view(F, C) + p[F * C:]).argmax(1) == y.long()).sum())
        assert abs(int(ref.item()) - expect) <= max(2, n // 2000)  # fp32 vs fp64 near-ties only
        for cap in (1, 8, 48, 0, 10_000):
            got = torch.zeros(1, dtype=torch.int64, device="cuda")
            _abi.check(_abi.lib.fedhc_eval_ctas(x.data_ptr(), y.data_ptr(), n, F, C, p.data_ptr(), got.data_ptr(),
                                                cap, st))
            assert int(got.item()) == int(ref.item()), (n, cap)


def test_accuracy_first_max_ties_class_groups():
    """The row kernel's 16-class groups (C <= 64): all-tied logits pick class 0 (np.argmax's first maximum),
    and a maximum in a later group or the last real class is found; padding classes never win."""
    import torch
    from paper_2305_15668_b200 import _abi
    g = torch.Generator(device="cuda").manual_seed(9)
    st = torch.cuda.current_stream().cuda_stream
    for C in (20, 40, 62, 64):
        F, n = 784, 777
        x = torch.randn(n, F, device="cuda", generator=g)
        y = torch.randint(0, C, (n,), device="cuda", generator=g, dtype=torch.int32)
        p = torch.zeros(F * C + C, device="cuda", dtype=torch.float64)
        got = torch.zeros(1, dtype=torch.int64, device="cuda")
        _abi.check(_abi.lib.fedhc_eval(x.data_ptr(), y.data_ptr(), n, F, C, p.data_ptr(), got.data_ptr(), st))
        assert int(got.item()) == int((y == 0).sum())
        for top in (C - 1, 17 % C, 33 % C):  # the bias alone decides: a single maximum at class `top`
            p.zero_()
            p[F * C + top] = 1.0
            got.zero_()
            _abi.check(_abi.lib.fedhc_eval(x.data_ptr(), y.data_ptr(), n, F, C, p.data_ptr(), got.data_ptr(), st))
            assert int(got.item()) == int((y == top).sum()), (C, top)


def test_loss_and_grad_vs_oracle(tr):
    loss, grad = tr.loss_and_grad(FL["lg_p"], FL["lg_x"], FL["lg_y"], 4)
    assert loss == pytest.approx(float(FL["lg_loss"]), rel=1e-12)
    assert rel_err(grad, FL["lg_grad"]) <= 1e-12
    rng = np.random.default_rng(1)
    loss, _ = tr.loss_and_grad(np.zeros(15), rng.standard_normal((50, 2)), rng.integers(0, 5, 50), 5)
    assert loss == pytest.approx(np.log(5))


def test_train_experiments_vs_golden(fh):
    tz = np.load(os.path.join(GOLDEN, "train_small.npz"))
    meta = json.loads(str(tz["meta"]))
    for i, m in enumerate(meta):
        fleet = fh.generate_fleet(fh.DistributionSpec(**m["fleet"]["spec"]), m["fleet"]["n"], m["fleet"]["seed"])
        rep = fh.run_experiment(fh.FleetConfig(**m["cfg"]), fleet, fh.DataParams(**m["data"]),
                                fh.TrainParams(enabled=True, lr=m["lr"]))
        assert rep.participants == m["participants"]
        assert rel_err(rep.final_params, tz[f"tr{i}_params"]) <= REL
        acc = np.array(rep.accuracy_series)
        want = tz[f"tr{i}_acc"]
        assert np.array_equal(acc[:, 0], want[:, 0])  # aggregation times: bit-exact DES
        assert np.max(np.abs(acc[:, 1] - want[:, 1])) <= 0.02


@pytest.mark.parametrize("classes", [10, 62])
def test_femnist_round_vs_golden(fh, classes):
    g = np.load(os.path.join(GOLDEN, f"round_c{classes}.npz"))
    fleet = fh.generate_fleet(fh.DistributionSpec(budget_levels=(10, 15, 30, 40, 50, 65, 80), num_samples=6400,
                                                  batch_size=64), 10, 1)
    rep = fh.run_experiment(fh.FleetConfig(participants_per_round=10, rounds=1, seed=1), fleet,
                            fh.DataParams(features=784, classes=classes, alpha=0.5), fh.TrainParams(True, 0.1))
    assert rep.participants[0] == list(g["participants"])
    assert rep.rounds[0].makespan == float(g["makespan"])
    err = rel_err(rep.final_params, g["params"])
    assert err <= REL, err
    assert abs(rep.accuracy_series[0][1] - float(g["acc"][0][1])) <= 2 / 16000


@pytest.mark.parametrize("C", [10, 62])
def test_batched_round_matches_per_client(fh, tr, C):
    """DeviceFederation.train (one launch, many clients) == per-client oracle local_train."""
    import torch
    from paper_2305_15668_b200.experiment import DeviceFederation
    from paper_2305_15668_b200.spec import WorkloadSpec
    trn, tst = fm.synthetic(784, C, 6000, seed=11)
    sizes = [640, 700, 0, 64, 1000, 333]
    shards, at = {}, 0
    for i, n in enumerate(sizes):
        shards[f"c{i}"] = tr.DatasetShard(f"c{i}", trn.features[at:at + n], trn.labels[at:at + n])
        at += n
    fed = DeviceFederation(shards, tr.Dataset(tst.features, tst.labels, C), 784, C)
    params = np.random.default_rng(2).standard_normal(784 * C + C) * 0.01
    wl = [WorkloadSpec(n if n else 10, 64) for n in sizes]
    seeds = [fm.seed_of("train", 1, 0, f"c{i}") for i in range(len(sizes))]
    p = torch.from_numpy(params).cuda()
    deltas = fed.train(p, list(shards), wl, 0.1, seeds).cpu().numpy()
    for i, cid in enumerate(shards):
        want = fm.local_sgd(params, fm.Shard(cid, shards[cid].features, shards[cid].labels), wl[i].num_samples,
                            wl[i].batch_size, 0.1, C, seed=seeds[i])
        if sizes[i] == 0:
            assert np.all(deltas[i] == 0)
        else:
            assert rel_err(deltas[i], want) <= REL


@pytest.mark.parametrize("F", [784, 720])
def test_c62_round_with_tail_wave(fh, tr, F):
    """More participants than 2-CTA clusters fit at once (74 on a B200: a second, partial wave): every client's
    delta (ragged and reshuffled batches, an empty shard) == the per-client oracle local_train.  F = 720: 11 chunks
    + a 16-feature tail (uneven CTAs)."""
    import torch
    from paper_2305_15668_b200.experiment import DeviceFederation
    from paper_2305_15668_b200.spec import WorkloadSpec
    C, K = 62, 96
    sizes = [96 + (i % 5) * 17 for i in range(K)]
    sizes[80] = 0
    trn, tst = fm.synthetic(F, C, sum(sizes) + 200, seed=5)
    shards, at = {}, 0
    for i, n in enumerate(sizes):
        shards[f"c{i}"] = tr.DatasetShard(f"c{i}", trn.features[at:at + n], trn.labels[at:at + n])
        at += n
    fed = DeviceFederation(shards, tr.Dataset(tst.features, tst.labels, C), F, C)
    params = np.random.default_rng(3).standard_normal(F * C + C) * 0.02
    wl = [WorkloadSpec(2 * n if n else 10, 64) for n in sizes]
    seeds = [fm.seed_of("train", 2, 0, f"c{i}") for i in range(K)]
    deltas = fed.train(torch.from_numpy(params).cuda(), list(shards), wl, 0.1, seeds).cpu().numpy()
    for i in list(range(0, K, 7)) + [73, 74, 75, 79, 80, K - 1]:
        cid = f"c{i}"
        if sizes[i] == 0:
            assert np.all(deltas[i] == 0)
            continue
        want = fm.local_sgd(params, fm.Shard(cid, shards[cid].features, shards[cid].labels), wl[i].num_samples,
                            wl[i].batch_size, 0.1, C, seed=seeds[i])
        assert rel_err(deltas[i], want) <= REL, (i, rel_err(deltas[i], want))


@pytest.mark.parametrize("F", [784, 720])
def test_c62_wrap_schedule_bit_identical(fh, tr, F):
    """More clients than resident 2-CTA clusters: train_c64_kernel lays the clients' steps out on the resident
    clusters by McNaughton's wrap-around rule, so a client cut at a slot boundary runs its first steps on one
    cluster, saves its state, and finishes on another.  Same steps, same order: the deltas must equal, bit for
    bit, the ones of launches small enough to run every client whole on one cluster."""
    import torch
    from paper_2305_15668_b200.experiment import DeviceFederation
    from paper_2305_15668_b200.spec import WorkloadSpec
    C, K = 62, 170
    sizes = [40 + (i * 37) % 150 for i in range(K)]
    sizes[9] = 0
    sizes[100] = 1
    trn, tst = fm.synthetic(F, C, sum(sizes) + 200, seed=6)
    shards, at = {}, 0
    for i, n in enumerate(sizes):
        shards[f"c{i}"] = tr.DatasetShard(f"c{i}", trn.features[at:at + n], trn.labels[at:at + n])
        at += n
    fed = DeviceFederation(shards, tr.Dataset(tst.features, tst.labels, C), F, C)
    params = torch.from_numpy(np.random.default_rng(4).standard_normal(F * C + C) * 0.02).cuda()
    wl = [WorkloadSpec(3 * n if n else 10, 64) for n in sizes]   # several reshuffles, ragged batches
    ids = list(shards)
    seeds = [fm.seed_of("train", 3, 0, c) for c in ids]
    whole = fed.train(params, ids, wl, 0.1, seeds).cpu().numpy()
    parts = [fed.train(params, ids[a:a + 40], wl[a:a + 40], 0.1, seeds[a:a + 40]).cpu().numpy()
             for a in range(0, K, 40)]
    cut = np.concatenate(parts)
    assert whole.shape == cut.shape
    bad = [i for i in range(K) if not np.array_equal(whole[i], cut[i])]
    assert not bad, bad[:10]
    assert np.all(whole[9] == 0)


def test_x_split_layout(fh):
    """fedhc_x_split: each row -> per 8-feature unit [8 bf16 hi | 8 bf16 mid], hi = bf16_rn(x),
    mid = bf16_rn(x - hi)."""
    import torch
    from paper_2305_15668_b200.training import x_split
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(37, 784, device="cuda", generator=g) * 3
    x[0, :4] = torch.tensor([0.0, -0.0, 1e-30, -7.5e5])
    got = x_split(x).view(torch.int16).view(37, 98, 2, 8)
    hi = x.to(torch.bfloat16)
    mid = (x - hi.float()).to(torch.bfloat16)
    assert torch.equal(got[:, :, 0].reshape(37, 784), hi.view(torch.int16))
    assert torch.equal(got[:, :, 1].reshape(37, 784), mid.view(torch.int16))


@pytest.mark.parametrize("sizes,b,lr", [
    ([640, 700, 0, 64, 1000, 333], 64, 0.1),   # ragged batches, reshuffles, an empty shard
    ([100, 17, 256], 16, 0.05),                 # one stage per batch, partial stages
    ([90, 1], 1, 0.1),                          # batch of one row
])
def test_split_rows_bit_identical(fh, tr, sizes, b, lr):
    """The split-row trainer (train_pipe2_kernel: fedhc_x_split copy, ldmatrix fragments, 12 balanced compute
    warps) vs the fp32-row trainer (train_pipe_kernel, splits in registers): the same bf16x3 products summed in
    a different grouping -> equal to fp32 rounding (<= 2e-6 of max|delta|); deterministic; both vs the oracle."""
    import torch
    from paper_2305_15668_b200 import _abi
    from paper_2305_15668_b200.experiment import DeviceFederation, delta_buffer
    from paper_2305_15668_b200.spec import WorkloadSpec
    from paper_2305_15668_b200.training import stream_ptr
    C = 10
    trn, tst = fm.synthetic(784, C, sum(sizes) + 10, seed=5)
    shards, at = {}, 0
    for i, n in enumerate(sizes):
        shards[f"c{i}"] = tr.DatasetShard(f"c{i}", trn.features[at:at + n], trn.labels[at:at + n])
        at += n
    fed = DeviceFederation(shards, tr.Dataset(tst.features, tst.labels, C), 784, C)
    assert fed.x_split is not None
    params = torch.from_numpy(np.random.default_rng(4).standard_normal(784 * C + C) * 0.01).cuda()
    wl = [WorkloadSpec(n if n else 10, b) for n in sizes]
    seeds = [fm.seed_of("train", 1, 0, f"c{i}") for i in range(len(sizes))]
    ids = list(shards)
    meta, _ = fed.stage_plan(ids, wl, seeds)
    d_split, d_f32 = delta_buffer(len(ids), fed.P, "cuda"), delta_buffer(len(ids), fed.P, "cuda")
    desc_a = fed.descriptors(ids, meta, lr, d_split)
    desc_b = fed.descriptors(ids, meta, lr, d_f32)
    fed.launch_train(desc_a.data_ptr(), len(ids), params, b)
    _abi.check(_abi.lib.fedhc_local_train(desc_b.data_ptr(), len(ids), params.data_ptr(), 784, C, b, stream_ptr()))
    torch.cuda.synchronize()
    scale = float(d_f32.abs().max())
    assert float((d_split - d_f32).abs().max()) <= 2e-6 * scale
    again = d_split.clone()
    fed.launch_train(desc_a.data_ptr(), len(ids), params, b)
    torch.cuda.synchronize()
    assert torch.equal(again, d_split)
    for i, cid in enumerate(ids):
        if sizes[i]:
            want = fm.local_sgd(params.cpu().numpy(), fm.Shard(cid, shards[cid].features, shards[cid].labels),
                                wl[i].num_samples, b, lr, C, seed=seeds[i])
            assert rel_err(d_split[i, :fed.P].cpu().numpy(), want) <= REL


def test_full_size_round_properties(fh):
    """Bench-size round (100 clients x 6400 x 784): finite deltas, determinism, FedAvg linearity."""
    import torch
    from paper_2305_15668_b200.experiment import DeviceFederation
    from paper_2305_15668_b200.spec import WorkloadSpec
    K, n, F, C = 100, 6400, 784, 10
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn(K * n, F, device="cuda", generator=g)
    y = torch.randint(0, C, (K * n,), device="cuda", generator=g, dtype=torch.int32)
    offs = {f"c{i:03d}": (i * n, n) for i in range(K)}
    fed = DeviceFederation.from_arrays(x, y, offs, x[:1000], y[:1000], C)
    params = torch.zeros(F * C + C, dtype=torch.float64, device="cuda")
    wl = [WorkloadSpec(n, 64)] * K
    seeds = list(range(K))
    d1 = fed.train(params, list(offs), wl, 0.1, seeds).clone()
    d2 = fed.train(params, list(offs), wl, 0.1, seeds)
    assert torch.isfinite(d1).all() and torch.equal(d1, d2)
    # per-client spot check against the oracle on two clients
    xs, ys = x[:2 * n].cpu().double().numpy(), y[:2 * n].cpu().numpy().astype(int)
    for i in range(2):
        want = fm.local_sgd(np.zeros(F * C + C), fm.Shard("c", xs[i * n:(i + 1) * n], ys[i * n:(i + 1) * n]), n, 64,
                            0.1, C, seed=seeds[i])
        assert rel_err(d1[i].cpu().numpy(), want) <= REL
    fed.aggregate(params, d1, [1.0] * K)
    mean = d1.double().mean(0)
    assert torch.allclose(params, mean, rtol=1e-12, atol=1e-15)


def test_device_fleet_data_partition(fh):
    from paper_2305_15668_b200.devicedata import DeviceFleetData
    ids = [f"c{i:04d}" for i in range(50)]
    sizes = [int(v) for v in np.random.default_rng(0).choice([16, 32, 64, 128, 256, 512, 1024], 50)]
    d = DeviceFleetData(ids, sizes, 64, 10, alpha=0.5, seed=5, n_test=1000)
    assert d.x.shape == (sum(sizes), 64) and d.y.shape == (sum(sizes),)
    y = d.y.cpu().numpy()
    for i, cid in enumerate(ids):
        o, n = d.offsets[cid]
        assert n == sizes[i]
        assert np.array_equal(np.bincount(y[o:o + n], minlength=10), d.counts[i])
    # features cluster around the class means
    x = d.x[:2000].double()
    err = (x - d.means[d.y[:2000].long()].double()).std().item()
    assert 0.9 < err < 1.1
    fed = d.federation()
    assert fed.n_test == 1000 and fed.P == 64 * 10 + 10


def test_green_partitions_confine_kernels(fh):
    from paper_2305_15668_b200.live import GreenPartitions
    parts = GreenPartitions(0, 8)
    assert parts.n_groups >= 2 and parts.sms_per_group >= 8
    a = parts.probe(0, 1)
    b = parts.probe(1, 2)
    assert 0 < len(a) <= parts.sms_per_group
    assert 0 < len(b) <= 2 * parts.sms_per_group
    assert not (a & b), (a, b)  # disjoint windows -> disjoint SMs


def _replay_live_on_oracle(trace, by_id, cfg, participants):
    """Feed the live round's real-time event order to the ORACLE executor manager (oracle/orchestration.Manager,
    executor_manager.py:81-238) and check that every launch the live round made is the oracle's decision."""
    m = oc.Manager(cfg.max_executors, cfg.scheduler_kind, cfg.theta, cfg.dynamic_parallelism)
    m.begin_round([(c, float(by_id[c].resource_budget)) for c in participants])
    launches = [(e["client"], e["executor"]) for e in trace if e["kind"] == "ClientLaunched"]
    expected = []

    def take(decisions):
        for (cid, _b, ex), _instr in decisions:
            expected.append((cid, ex))
            m.request(cid, "register", 0.0)

    take(m.kickoff(0.0))
    for e in trace:
        if e["kind"] == "SlotFreed":
            m.request(e["client"], "training_complete", 0.0)
            m.request(e["client"], "model_uploaded", 0.0)
            take(m.slot_freed(e["executor"], 0.0))
    assert launches == expected
    return launches


def test_live_round_vs_oracle(fh, tr):
    """Real-time dispatch on green-context partitions (comms.py:94-457 semantics): every launch decision equals
    the oracle executor manager's under the same completion order, the deltas equal the batched launch's bit for
    bit, and the aggregated params match the oracle's fp64 round (local_sgd + FedAvg) within the bar."""
    import torch
    from paper_2305_15668_b200.experiment import DeviceFederation
    from paper_2305_15668_b200.live import GreenPartitions, LiveRound
    F, C = 784, 10
    fleet = fh.generate_fleet(fh.DistributionSpec(budget_levels=(10, 15, 30, 40, 50, 65, 80), num_samples=[320, 640],
                                                  batch_size=64), 12, 3)
    by_id = {p.client_id: p for p in fleet}
    trn, tst = fm.synthetic(F, C, 12000, seed=1)
    shards, at = {}, 0
    for p in fleet:
        n = p.workload.num_samples
        shards[p.client_id] = tr.DatasetShard(p.client_id, trn.features[at:at + n], trn.labels[at:at + n])
        at += n
    fed = DeviceFederation(shards, tr.Dataset(tst.features, tst.labels, C), F, C)
    cfg = fh.FleetConfig(participants_per_round=12, max_executors=6, seed=3)
    who = sorted(by_id)
    params = torch.zeros(F * C + C, dtype=torch.float64, device="cuda")
    live = LiveRound(fed, by_id, cfg, 0.1, GreenPartitions(0, 8))
    d_live, rep, trace, measured = live.run(params, who, round_index=0)
    seeds = [fm.seed_of("train", cfg.seed, 0, c) for c in who]
    d_batch = fed.train(params, who, [by_id[c].workload for c in who], 0.1, seeds)
    assert torch.equal(d_live, d_batch)
    assert set(measured) == set(who) and all(v > 0 for v in measured.values())
    assert rep.makespan > 0 and len(rep.per_client_end) == len(who)
    assert sorted(c for c, _ in _replay_live_on_oracle(trace, by_id, cfg, who)) == who
    live.aggregate(params, d_live, who)
    deltas = [fm.local_sgd(np.zeros(F * C + C), fm.Shard(c, shards[c].features, shards[c].labels),
                           by_id[c].workload.num_samples, 64, 0.1, C, seed=seeds[i]) for i, c in enumerate(who)]
    want = fm.weighted_average(deltas, [float(by_id[c].workload.num_samples) for c in who], np.zeros(F * C + C))
    assert rel_err(params.cpu().numpy(), want) <= REL


def test_live_cnn_round_budgets_are_physical(fh, tr):
    """FEMNIST-CNN clients (config 2's model) in the live mode: each client runs its own engine on the SM window
    its budget buys.  Deltas equal the batched engine's; launches follow the oracle manager; a 10 %-budget client
    (1 SM group) takes longer than a 80 %-budget client (several groups) for the same work."""
    import torch
    from paper_2305_15668_b200.cnn import CnnEngine, CnnFederation, init_cnn_params
    from paper_2305_15668_b200.live import GreenPartitions, LiveRound
    fleet = fh.generate_fleet(fh.DistributionSpec(budget_levels=(10, 80), num_samples=128, batch_size=64), 6, 5)
    by_id = {p.client_id: p for p in fleet}
    trn, tst = fm.synthetic(784, 10, 2000, seed=3)
    shards, at = {}, 0
    for p in fleet:
        shards[p.client_id] = tr.DatasetShard(p.client_id, trn.features[at:at + 128], trn.labels[at:at + 128])
        at += 128
    fed = CnnFederation(shards, tr.Dataset(tst.features, tst.labels, 10), 784, 10).attach_engine(6, 64)
    cfg = fh.FleetConfig(participants_per_round=6, max_executors=3, seed=5)
    who = sorted(by_id)
    params = torch.tensor(fed.layout.to_padded(init_cnn_params(10, 1)), dtype=torch.float64, device="cuda")
    parts = GreenPartitions(0, 8)
    engines = [CnnEngine(1, 64, 10) for _ in range(cfg.max_executors)]
    live = LiveRound(fed, by_id, cfg, 0.01, parts, engines=engines)
    live.run(params, who, round_index=0)      # warm-up (plans, module load)
    d_live, rep, trace, measured = live.run(params, who, round_index=0)
    seeds = [fm.seed_of("train", cfg.seed, 0, c) for c in who]
    d_batch = fed.train(params, who, [by_id[c].workload for c in who], 0.01, seeds, use_graph=False)
    assert torch.allclose(d_live, d_batch, rtol=0, atol=1e-6 * float(d_batch.abs().max()))
    _replay_live_on_oracle(trace, by_id, cfg, who)
    lo = [measured[c] for c in who if by_id[c].resource_budget == 10]
    hi = [measured[c] for c in who if by_id[c].resource_budget == 80]
    assert lo and hi and min(lo) > max(hi), (lo, hi)


@pytest.mark.parametrize("G,M,N,K", [(1, 128, 128, 64), (3, 256, 384, 512), (5, 2048, 128, 3136 // 64 * 64),
                                     (2, 256, 512, 1024), (7, 384, 256, 3136 // 64 * 64)])
def test_tcgen05_grouped_gemm_vs_torch(fh, G, M, N, K):
    """tcgen05 grouped GEMM (bf16 in, fp32 accumulate) vs torch fp32 on the same bf16 values."""
    import torch
    from paper_2305_15668_b200 import _abi
    g = torch.Generator(device="cuda").manual_seed(G * 7 + M)
    A = torch.randn(G, M, K, device="cuda", generator=g).to(torch.bfloat16)
    B = torch.randn(G, N, K, device="cuda", generator=g).to(torch.bfloat16)
    D = torch.full((G, M, N), float("nan"), device="cuda")
    _abi.check(_abi.lib.fedhc_gemm_bf16_tn(G, M, N, K, A.data_ptr(), B.data_ptr(), D.data_ptr(),
                                           torch.cuda.current_stream().cuda_stream))
    ref = torch.bmm(A.float(), B.float().transpose(1, 2))
    assert torch.isfinite(D).all()
    err = (D - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-5, err


@pytest.mark.parametrize("a_mn,b_mn", [(False, False), (True, False), (False, True), (True, True)])
@pytest.mark.parametrize("G,M,N,K", [(1, 128, 64, 64), (3, 256, 192, 320), (2, 128, 256, 1024), (4, 384, 128, 128),
                                     (3, 64, 64, 2048), (2, 64, 2048, 64), (5, 192, 96, 128), (2, 64, 32, 512),
                                     (3, 256, 32, 64), (2, 128, 576, 64), (2, 64, 960, 128)])
def test_gemm_operand_majors_vs_torch(fh, a_mn, b_mn, G, M, N, K):
    """Every operand storage (K- or MN-major) and N tile (64/128/256) against torch fp32."""
    import torch
    from paper_2305_15668_b200.gemm import gemm
    if b_mn and N % 64:
        pytest.skip("N=32 tiles take a K-major B only")
    g = torch.Generator(device="cuda").manual_seed(G * 1000 + M + N + K + 2 * a_mn + b_mn)
    A = torch.randn(G, M, K, device="cuda", generator=g).to(torch.bfloat16)
    B = torch.randn(G, N, K, device="cuda", generator=g).to(torch.bfloat16)
    ref = torch.bmm(A.float(), B.float().transpose(1, 2))
    a_op = A.transpose(1, 2).contiguous() if a_mn else A
    b_op = B.transpose(1, 2).contiguous() if b_mn else B
    D = gemm(a_op, b_op, a_mn=a_mn, b_mn=b_mn)
    err = (D - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-5, err


@pytest.mark.parametrize("per_row", [False, True])
def test_gemm_bias_relu_bf16_epilogue(fh, per_row):
    import torch
    from paper_2305_15668_b200.gemm import EPI_BF16, EPI_BIAS_RELU_BF16, gemm
    G, M, N, K = 2, 256, 192, 256
    g = torch.Generator(device="cuda").manual_seed(11 + per_row)
    A = torch.randn(G, M, K, device="cuda", generator=g).to(torch.bfloat16)
    B = torch.randn(G, N, K, device="cuda", generator=g).to(torch.bfloat16)
    bias = torch.randn(G, M if per_row else N, device="cuda", generator=g)
    acc = torch.bmm(A.float(), B.float().transpose(1, 2))
    ref = torch.relu(acc + (bias[:, :, None] if per_row else bias[:, None, :]))
    D = gemm(A, B, epilogue=EPI_BIAS_RELU_BF16, bias=bias, bias_per_row=per_row)
    # bf16 rounding (2^-8 relative) of fp32 values that differ only in accumulation order
    tol = ref.abs() * 2 ** -8 + 1e-5 * acc.abs().max()
    assert ((D.float() - ref).abs() <= tol).all()
    D2 = gemm(A, B, epilogue=EPI_BF16)
    assert ((D2.float() - acc).abs() <= acc.abs() * 2 ** -8 + 1e-5 * acc.abs().max()).all()


def test_gemm_sgd_epilogue_in_place(fh):
    """master -= lr * (A . B^T) in place, bf16 shadow == master rounded."""
    import torch
    from paper_2305_15668_b200.gemm import EPI_SGD, gemm
    G, M, N, K = 3, 128, 320, 512
    g = torch.Generator(device="cuda").manual_seed(5)
    A = torch.randn(G, K, M, device="cuda", generator=g).to(torch.bfloat16)   # MN-major, like a wgrad
    B = torch.randn(G, K, N, device="cuda", generator=g).to(torch.bfloat16)
    W = torch.randn(G, M, N, device="cuda", generator=g)
    ref = W - 0.01 * torch.bmm(A.float().transpose(1, 2), B.float())
    shadow = torch.empty(G, M, N, dtype=torch.bfloat16, device="cuda")
    gemm(A, B, a_mn=True, b_mn=True, epilogue=EPI_SGD, master=W, shadow=shadow, lr=0.01)
    assert (W - ref).abs().max().item() < 1e-5 * ref.abs().max().item() + 1e-6
    assert torch.equal(shadow, W.to(torch.bfloat16))


@pytest.mark.parametrize("M,N", [(2048, 64), (64, 64), (128, 32)])
def test_gemm_relu_mask_rowsum_epilogue(fh, M, N):
    """ReLU backward fused in the epilogue: D = acc * (mask > 0), rowsum = sum_n D (bias gradient)."""
    import torch
    from paper_2305_15668_b200.gemm import EPI_RELU_MASK_BF16, gemm
    G, K = 3, 128
    g = torch.Generator(device="cuda").manual_seed(M + N)
    A = torch.randn(G, K, M, device="cuda", generator=g).to(torch.bfloat16)
    B = torch.randn(G, N, K, device="cuda", generator=g).to(torch.bfloat16)
    mask = torch.relu(torch.randn(G, M, N, device="cuda", generator=g)).to(torch.bfloat16)
    acc = torch.bmm(A.float().transpose(1, 2), B.float().transpose(1, 2))
    ref = acc * (mask > 0)
    rs = torch.full((G, M), float("nan"), device="cuda")
    D = gemm(A, B, a_mn=True, epilogue=EPI_RELU_MASK_BF16, mask=mask, rowsum=rs)
    assert ((D.float() - ref).abs() <= ref.abs() * 2 ** -8 + 1e-5 * acc.abs().max()).all()
    assert torch.equal(D == 0, ref.to(torch.bfloat16) == 0) or ((D == 0) != (ref == 0)).sum() < 4
    assert torch.allclose(rs, D.float().sum(-1), rtol=1e-5, atol=1e-4)


def test_gemm_rejects_bad_shapes(fh):
    import torch
    from paper_2305_15668_b200.gemm import gemm
    A = torch.zeros(1, 100, 64, dtype=torch.bfloat16, device="cuda")
    B = torch.zeros(1, 64, 64, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(NotImplementedError):
        gemm(A, B)


def test_device_permutations_match_numpy(fh):
    import torch
    from paper_2305_15668_b200 import _abi
    seeds = [5, 99, 123456, 4294967295, 0, 31337, 7]
    rows = [6400, 1, 77, 1000, 2, 300, 70000]   # last one permutes in global memory
    perms = [1, 3, 2, 1, 4, 2, 1]
    sizes = np.array(rows, np.int64) * np.array(perms, np.int64)
    offs = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
    dev = lambda a, t: torch.from_numpy(np.ascontiguousarray(a, dtype=t)).cuda()  # noqa: E731
    s_d, r_d, p_d, o_d = dev(seeds, np.uint64), dev(rows, np.int32), dev(perms, np.int32), dev(offs, np.int64)
    out = torch.full((int(sizes.sum()),), -1, dtype=torch.int32, device="cuda")
    _abi.check(_abi.lib.fedhc_batch_permutations_device(s_d.data_ptr(), r_d.data_ptr(), p_d.data_ptr(), o_d.data_ptr(),
                                                        len(seeds), out.data_ptr(), max(rows[:-1]),
                                                        torch.cuda.current_stream().cuda_stream))
    got = out.cpu().numpy()
    for s, n, k, o in zip(seeds, rows, perms, offs):
        g = np.random.default_rng(s)
        assert np.array_equal(got[o:o + n * k], np.concatenate([g.permutation(n) for _ in range(k)]))


@pytest.mark.parametrize("legacy", [False, True])
def test_device_permutations_sizes_sweep(fh, legacy, monkeypatch):
    """perm_fast_kernel (parallel acceptance scan + bucket chains) and the sequential walk vs numpy, at sizes
    around powers of two (mask changes), tiny shards and several permutations per client."""
    import subprocess
    import sys
    code = f"""
import numpy as np, torch
from paper_2305_15668_b200 import _abi
rng = np.random.default_rng(11)
rows = [1, 2, 3, 31, 32, 33, 63, 64, 65, 127, 128, 129, 1023, 1024, 1025, 4095, 4096, 4097, 6400, 8191, 5000]
perms = [int(rng.integers(1, 4)) for _ in rows]
seeds = [int(x) for x in rng.integers(0, 2**32, len(rows))]
sizes = np.array(rows, np.int64) * np.array(perms, np.int64)
offs = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
dev = lambda a, t: torch.from_numpy(np.ascontiguousarray(a, dtype=t)).cuda()
s_d, r_d, p_d, o_d = dev(seeds, np.uint64), dev(rows, np.int32), dev(perms, np.int32), dev(offs, np.int64)
out = torch.full((int(sizes.sum()),), -1, dtype=torch.int32, device="cuda")
_abi.check(_abi.lib.fedhc_batch_permutations_device(s_d.data_ptr(), r_d.data_ptr(), p_d.data_ptr(), o_d.data_ptr(),
           len(seeds), out.data_ptr(), 6400, torch.cuda.current_stream().cuda_stream))
got = out.cpu().numpy()
for s, n, k, o in zip(seeds, rows, perms, offs):
    g = np.random.default_rng(s)
    assert np.array_equal(got[o:o + n * k], np.concatenate([g.permutation(n) for _ in range(k)])), (n, k)
print("ok")
"""
    env = dict(os.environ)
    if legacy:
        env["FEDHC_PERM_LEGACY"] = "1"
    res = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                         cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert res.returncode == 0 and "ok" in res.stdout, res.stderr[-2000:]


def test_runner_device_plan_matches_host_plan(fh):
    """FederatedRunner with GPU-generated batch order == host-generated order, and CUDA-graph replay == eager
    launches, bit for bit, over 4 rounds (graphs are captured at a slot's first use, replayed after)."""
    import torch
    from paper_2305_15668_b200.devicedata import DeviceFleetData
    from paper_2305_15668_b200.experiment import FederatedRunner
    fleet = fh.generate_fleet(fh.DistributionSpec(budget_levels=(10, 30, 50, 80), num_samples=[320, 640, 700],
                                                  batch_size=[32, 64]), 24, 9)
    by_id = {p.client_id: p for p in fleet}
    ids = sorted(by_id)
    data = DeviceFleetData(ids, [by_id[c].workload.num_samples for c in ids], 784, 10, 0.5, seed=3, n_test=2000)
    cfg = fh.FleetConfig(participants_per_round=16, max_executors=8, seed=9)
    outs = []
    # host plan, device plan (native round loop, the default), device plan through the Python launch path,
    # device plan replayed from per-slot CUDA graphs
    for device_perm, graphs, native in ((False, False, False), (True, False, True), (True, False, False),
                                        (True, True, False)):
        params = torch.zeros(7850, dtype=torch.float64, device="cuda")
        r = FederatedRunner(data.federation(), by_id, cfg, 0.1, params=params, device_permutations=device_perm,
                            use_graphs=graphs, native=native)
        assert (r._native is not None) == native
        series = r.run(4)
        outs.append((params.clone(), series))
    # the same 4 rounds as run(1) + run(3): each call plans the next call's first round while draining
    params = torch.zeros(7850, dtype=torch.float64, device="cuda")
    r = FederatedRunner(data.federation(), by_id, cfg, 0.1, params=params)
    outs.append((None, r.run(1) + r.run(3)))
    outs[-1] = (params.clone(), outs[-1][1])
    for o in outs[1:]:
        assert torch.equal(outs[0][0], o[0])
        assert outs[0][1] == o[1]


def test_runner_async_native_matches_python_path(fh):
    """Async aggregation (engine.py:354-364) in the native round loop (chunked FedAvg on the params, per-chunk
    snapshots evaluated on the side stream) == the Python launch path (per-chunk FedAvg + accuracy in stream
    order), bit for bit, and run(1) + run(2) == run(3)."""
    import torch
    from paper_2305_15668_b200.devicedata import DeviceFleetData
    from paper_2305_15668_b200.experiment import FederatedRunner
    fleet = fh.generate_fleet(fh.DistributionSpec(budget_levels=(10, 30, 50, 80), num_samples=[320, 640, 700],
                                                  batch_size=[32, 64]), 24, 4)
    by_id = {p.client_id: p for p in fleet}
    ids = sorted(by_id)
    data = DeviceFleetData(ids, [by_id[c].workload.num_samples for c in ids], 784, 10, 0.5, seed=3, n_test=2000)
    outs = []
    for native, buf, split_calls in ((True, 3, False), (False, 3, False), (True, 3, True), (True, 16, False)):
        cfg = fh.FleetConfig(participants_per_round=16, max_executors=8, seed=4, aggregation="async",
                             async_buffer=buf)
        params = torch.zeros(7850, dtype=torch.float64, device="cuda")
        r = FederatedRunner(data.federation(), by_id, cfg, 0.1, params=params, native=native)
        assert (r._native is not None) == native
        series = r.run(1) + r.run(2) if split_calls else r.run(3)
        assert len(series) == 3 * -(-16 // buf)
        outs.append((params.clone(), series, r.now))
    for o in outs[1:3]:
        assert torch.equal(outs[0][0], o[0]) and outs[0][1] == o[1] and outs[0][2] == o[2]
    assert outs[3][2] == outs[0][2]  # one chunk of all 16: the same DES times


@pytest.mark.parametrize("a_mn", [False, True])
def test_gemm_strided_operands_vs_torch(fh, a_mn):
    """Row strides (fedhc_gemm_args.lda / ldd): A read as a column slice of a wider row-major tensor (the
    ShuffleNetV2 engine's split-form X2 view) and D written into a column slice of a wider output."""
    import ctypes as C
    import torch
    from paper_2305_15668_b200 import _abi
    G, M, N, K, wide = 3, 256, 128, 64, 192
    g = torch.Generator(device="cuda").manual_seed(7 + int(a_mn))
    B = torch.randn(G, N, K, device="cuda", generator=g).to(torch.bfloat16)
    if a_mn:  # A stored [G][K][wide] MN-major, the GEMM reads columns [64, 64 + M') of each row
        Mw = 64
        big = torch.randn(G, K, wide, device="cuda", generator=g).to(torch.bfloat16)
        A_view, lda, Mv = big[:, :, 64:64 + Mw], wide, Mw
        ref = torch.bmm(A_view.float().transpose(1, 2), B.float().transpose(1, 2))
        a_ptr = big.data_ptr() + 64 * 2
    else:     # A stored [G][M][wide] K-major, the GEMM reads columns [64, 128)
        big = torch.randn(G, M, wide, device="cuda", generator=g).to(torch.bfloat16)
        A_view, lda, Mv = big[:, :, 64:64 + K], wide, M
        ref = torch.bmm(A_view.float(), B.float().transpose(1, 2))
        a_ptr = big.data_ptr() + 64 * 2
    Dbig = torch.zeros(G, Mv, N + 64, dtype=torch.bfloat16, device="cuda")
    args = _abi.GemmArgs(G=G, M=Mv, N=N, K=K, a_mn=int(a_mn), b_mn=0, A=a_ptr, B=B.data_ptr(),
                         epilogue=1, D=Dbig.data_ptr() + 64 * 2, ldd=N + 64, lda=lda,
                         a_gstride=big.shape[1] * wide)
    _abi.check(_abi.lib.fedhc_gemm(C.byref(args), torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    got = Dbig[:, :, 64:].float()
    err = (got - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-2, err
    assert not Dbig[:, :, :64].any()  # columns outside the view untouched
