"""Pin the CPU oracle against the reference's golden vectors (CPU only).

The fixtures in tests/golden/ were produced by running the real reference
(`tests/golden/make_golden.py`); the known-answer cases below are the
reference's own tests (pkg/tests/test_fl_core.py, test_scheduler.py,
test_engine.py, test_acceptance.py) restated.
"""

import json
import os
from collections import deque

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import flmath as fm
from oracle import orchestration as oc

FL = np.load(os.path.join(GOLDEN, "flcore.npz"))
with open(os.path.join(GOLDEN, "orchestration.json")) as fh:
    ORCH = json.load(fh)


def golden_fleets():
    import importlib.util
    spec = importlib.util.spec_from_file_location("mg", os.path.join(GOLDEN, "make_golden.py"))
    mg = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mg)
    return mg


MG = golden_fleets()


def oracle_fleet(case):
    return oc.fleet(case["n"], case["seed"], **case["spec"])


def rows_of(fleet):
    return [[c.client_id, c.resource_budget, c.workload.num_samples, c.workload.batch_size,
             c.workload.model_layers, c.workload.seq_len, c.workload.extra_model_factor,
             [list(p) for p in c.phases]] for c in fleet]


# -- fl_core ----------------------------------------------------------------


def test_stable_seed():
    parts = [("train", 1, 0, "c0000"), ("data", 1), ("partition", 1), ("local_train", 123), ("x",),
             ("train", 9, 3, "A")]
    assert [fm.seed_of(*p) for p in parts] == [int(v) for v in FL["seeds"]]


def test_dataset_bit_exact():
    tr, te = fm.synthetic(5, 3, 200, seed=42)
    assert np.array_equal(tr.features, FL["ds_train_x"]) and np.array_equal(tr.labels, FL["ds_train_y"])
    assert np.array_equal(te.features, FL["ds_test_x"]) and np.array_equal(te.labels, FL["ds_test_y"])


def test_dataset_edge_cases():
    tr, te = fm.synthetic(2, 3, 0, seed=1)
    assert len(tr.labels) == 0 and len(te.labels) == 0
    with pytest.raises(ValueError):
        fm.synthetic(0, 3, 10, seed=1)
    with pytest.raises(ValueError):
        fm.synthetic(2, 1, 10, seed=1)


def test_partition_bit_exact():
    tr, _ = fm.synthetic(3, 4, 2000, seed=5)
    clients = [(f"k{i}", n) for i, n in enumerate([100, 250, 17, 0, 400])]
    shards = fm.dirichlet_partition(tr, clients, 0.3, seed=11)
    for cid, n in clients:
        assert np.array_equal(shards[cid].labels, FL[f"part_{cid}_y"])
        assert np.array_equal(shards[cid].features, FL[f"part_{cid}_x"])
        assert len(shards[cid].labels) == n
    with pytest.raises(ValueError, match="want"):
        fm.dirichlet_partition(tr, [("a", 10**6)], 0.5, seed=1)
    with pytest.raises(ValueError):
        fm.dirichlet_partition(tr, [("a", 10)], 0.0, seed=1)


def test_loss_and_grad():
    loss, grad = fm.ce_grad(FL["lg_p"], FL["lg_x"], FL["lg_y"], 4)
    assert loss == float(FL["lg_loss"])
    assert np.array_equal(grad, FL["lg_grad"])


def test_gradient_vs_finite_difference():
    # pkg/tests/test_fl_core.py:125-134
    rng = np.random.default_rng(0)
    x = rng.standard_normal((20, 3))
    y = rng.integers(0, 4, size=20)
    p = rng.standard_normal(16) * 0.5
    _, g = fm.ce_grad(p, x, y, 4)
    num = np.zeros_like(p)
    for i in range(len(p)):
        e = np.zeros_like(p)
        e[i] = 1e-6
        num[i] = (fm.ce_grad(p + e, x, y, 4)[0] - fm.ce_grad(p - e, x, y, 4)[0]) / 2e-6
    assert np.max(np.abs(g - num) / np.maximum(np.abs(num), 1e-8)) < 1e-4


def test_zero_params_loss_is_log_c():
    rng = np.random.default_rng(1)
    loss, _ = fm.ce_grad(fm.zeros_params(2, 5), rng.standard_normal((50, 2)), rng.integers(0, 5, 50), 5)
    assert loss == pytest.approx(np.log(5))


@pytest.mark.parametrize("i", range(6))
def test_local_train_bit_exact(i):
    F, C, n, ns, b, lr = FL["lt_cases"][i]
    F, C, n, ns, b = int(F), int(C), int(n), int(ns), int(b)
    sd = str(FL["lt_seeds"][i])
    seed = int(sd) if sd.lstrip("-").isdigit() else sd
    shard = fm.Shard("a", FL[f"lt{i}_x"], FL[f"lt{i}_y"])
    d = fm.local_sgd(FL[f"lt{i}_p"], shard, ns, b, float(lr), C, seed=seed)
    assert np.array_equal(d, FL[f"lt{i}_d"])


def test_fedavg_goldens():
    # pkg/tests/test_fl_core.py:178-200
    base = np.array([1.0, 1.0])
    ds = [np.array([2.0, 4.0]), np.array([4.0, 6.0])]
    assert fm.weighted_average(ds, [1.0, 1.0], base) == pytest.approx([4.0, 6.0])
    assert fm.weighted_average(ds, [3.0, 1.0], base) == pytest.approx([3.5, 5.5])
    assert np.array_equal(fm.weighted_average([np.zeros(2)] * 2, [1.0, 2.0], np.array([1.5, -2.0])),
                          np.array([1.5, -2.0]))
    for args in ([], []), ([np.zeros(2)], [1.0, 2.0]), ([np.zeros(3)], [1.0]), ([np.zeros(2)], [0.0]), \
            ([np.zeros(2)], [-1.0]):
        with pytest.raises(fm.AggregationError):
            fm.weighted_average(args[0], args[1], np.zeros(2))
    out = fm.weighted_average(list(FL["fa_deltas"]), list(FL["fa_w"]), FL["fa_base"])
    assert np.array_equal(out, FL["fa_out"])


def test_accuracy():
    d = fm.Data(FL["acc_x"], FL["acc_y"], 6)
    assert fm.accuracy(FL["acc_p"], d) == float(FL["acc"])
    assert fm.accuracy(FL["acc_p"], fm.Data(np.zeros((0, 7)), np.zeros(0, int), 6)) == 0.0


# -- orchestration ------------------------------------------------------------


def test_fleets_bit_exact():
    for case, want in zip(MG.FLEET_CASES, ORCH["fleets"]):
        assert rows_of(oracle_fleet(case)) == want["rows"]


def test_case_study_schedules():
    pend = [(chr(65 + i), float(b)) for i, b in enumerate(oc.CASE_STUDY)]
    st = oc.SchedState(executors=range(8))
    assert [list(e) for e in oc.pick_resource_aware(st, pend, 8, 100.0)] == ORCH["case_study"]["ra"]
    assert st.total() == 100.0
    st = oc.SchedState(executors=range(8))
    assert [list(e) for e in oc.pick_greedy(st, pend, 8, 100.0)] == ORCH["case_study"]["greedy"]
    assert st.total() == 55.0


def test_scheduler_calls():
    for c in ORCH["sched_calls"]:
        st = oc.SchedState(c["running"], c["planned"], range(c["executors"]))
        got = oc.POLICIES[c["kind"]](st, [tuple(p) for p in c["pending"]], c["target"], c["theta"])
        assert [list(e) for e in got] == c["out"]
        assert [st.running, st.planned, list(st.free)] == c["state_after"]


def test_water_fill_and_work():
    for caps, dem, want in ORCH["maxmin"]:
        assert oc.water_fill(caps, dem) == want
    for (ns, b, l, s, x), want in ORCH["work"]:
        assert oc.work_of(oc.Workload(ns, b, l, s, x), 2e-6, 1e-3) == want


def _des_case(entry):
    fleets = [oracle_fleet(c) for c in MG.FLEET_CASES]
    fleet = {c.client_id: c for c in fleets[entry["fleet"]]}
    rep, seg = oc.simulate_round(fleet, entry["participants"], oc.Config(**entry["cfg"]))
    return rep, seg


def _norm(obj):
    return json.loads(json.dumps(obj, sort_keys=True))


def test_des_traces_bit_exact():
    for entry in ORCH["des"]:
        rep, seg = _des_case(entry)
        assert _norm(seg) == entry["trace"]
        assert _norm(rep) == entry["report"]


def test_selection_streams():
    import random
    for s in ORCH["selection"]:
        r = random.Random(f"{s['seed']}:selection")
        ids = [f"c{i:04d}" for i in range(120)]
        assert [r.sample(ids, 10) for _ in range(5)] == s["picks"]


def test_experiments_without_training():
    fleets = [oracle_fleet(c) for c in MG.FLEET_CASES]
    for entry in ORCH["experiments"]:
        trace = []
        out = oc.experiment(oc.Config(**entry["cfg"]), fleets[entry["fleet"]], trace=trace)
        assert out["participants"] == entry["participants"]
        assert _norm(out["rounds"]) == entry["rounds"]
        assert out["total_time"] == entry["total_time"]
        assert len(trace) == entry["trace_len"]
        assert _norm(trace[-40:]) == entry["trace_tail"]


def test_closed_form_des():
    # pkg/tests/test_engine.py:62-104 (unit workload: work == cfg.alpha)
    unit = oc.Workload(1, 1, 1, 1)
    mk = lambda bs, ph=((1.0, 100.0),): {f"c{i}": oc.Client(f"c{i}", b, unit, ph) for i, b in enumerate(bs)}
    cfg = lambda **kw: oc.Config(**{**dict(alpha=100.0, beta=0.0, max_executors=16), **kw})
    rep, _ = oc.simulate_round(mk([50, 25]), ["c0", "c1"], cfg())
    assert rep["per_client_times"] == pytest.approx({"c0": 200.0, "c1": 400.0})
    rep, _ = oc.simulate_round(mk([80, 65]), ["c0", "c1"], cfg())
    assert rep["makespan"] == pytest.approx(100 / 0.65 + 100 / 0.80)
    rep, _ = oc.simulate_round(mk([80, 65]), ["c0", "c1"], cfg(theta=150.0))
    assert rep["makespan"] == pytest.approx(200.0)
    rep, _ = oc.simulate_round(mk([50, 40, 30]), ["c0", "c1", "c2"], cfg(theta=150.0))
    assert rep["per_client_end"]["c0"] == pytest.approx(2000 / 7)
    assert rep["per_client_end"]["c2"] == pytest.approx(1000 / 3)
    rep, _ = oc.simulate_round(mk([50], oc.parse_phases("0.7:90;0.3:20")), ["c0"], cfg())
    assert rep["makespan"] == pytest.approx(70 / 0.5 + 30 / 0.2)
    rep, _ = oc.simulate_round(mk([10, 10, 10]), ["c0", "c1", "c2"], cfg(max_executors=1))
    assert rep["makespan"] == pytest.approx(3000.0)


def test_train_experiments_bit_exact():
    tz = np.load(os.path.join(GOLDEN, "train_small.npz"))
    meta = json.loads(str(tz["meta"]))
    for i, m in enumerate(meta):
        f = oc.fleet(m["fleet"]["n"], m["fleet"]["seed"], **m["fleet"]["spec"])
        out = oc.experiment(oc.Config(**m["cfg"]), f, train=True, lr=m["lr"], **m["data"])
        assert out["participants"] == m["participants"]
        assert np.array_equal(out["final_params"], tz[f"tr{i}_params"])
        assert np.array_equal(np.array(out["accuracy_series"]), tz[f"tr{i}_acc"])


@pytest.mark.parametrize("classes", [10, 62])
def test_femnist_round_bit_exact(classes):
    g = np.load(os.path.join(GOLDEN, f"round_c{classes}.npz"))
    f = oc.fleet(10, 1, budget_levels=(10, 15, 30, 40, 50, 65, 80), num_samples=6400, batch_size=64)
    out = oc.experiment(oc.Config(participants_per_round=10, rounds=1, seed=1), f, features=784,
                        classes=classes, alpha=0.5, train=True, lr=0.1)
    assert out["participants"][0] == list(g["participants"])
    assert np.array_equal(out["final_params"], g["params"])
    assert np.array_equal(np.array(out["accuracy_series"]), g["acc"])


@pytest.mark.parametrize("name", ["headline_rounds.npz", "headline_rounds_lr1e-3.npz"])
def test_headline_rounds_bit_exact(name):
    """bench.py's round shape at 640 samples/client: the oracle reproduces the reference's 10 rounds (final
    params, accuracy series, participants, makespans) bit for bit."""
    g = np.load(os.path.join(GOLDEN, name))
    h = json.loads(str(g["meta"]))
    f = oc.fleet(h["n"], h["seed"], budget_levels=tuple(h["budgets"]), num_samples=h["num_samples"],
                 batch_size=h["batch"])
    out = oc.experiment(oc.Config(participants_per_round=h["participants"], rounds=h["rounds"], seed=h["seed"],
                                  theta=h["theta"], max_executors=h["max_executors"]), f, features=h["features"],
                        classes=h["classes"], alpha=0.5, train=True, lr=h["lr"])
    assert out["participants"] == [list(p) for p in g["participants"]]
    assert [r["makespan"] for r in out["rounds"]] == g["makespans"].tolist()
    assert np.array_equal(out["final_params"], g["params"][-1])
    assert np.array_equal(np.array(out["accuracy_series"]), g["acc"])


def test_a8_runs_bit_exact():
    """Acceptance criterion A8's convergence runs (reference pkg/tests/test_acceptance.py:300-336)."""
    g = np.load(os.path.join(GOLDEN, "a8.npz"))

    def fleet_of(n, budgets, factor=1.0, samples=100):
        return [oc.Client(f"c{i:02d}", budgets[i % len(budgets)],
                          oc.Workload(num_samples=samples, batch_size=50, extra_model_factor=factor))
                for i in range(n)]

    for seed in (0, 3):
        for name, fl, k, rounds in (("wide", fleet_of(40, [10]), 20, 6), ("heavy", fleet_of(20, [50], 2.0), 10, 8),
                                    ("hetero", fleet_of(20, [10, 15, 30, 50, 80]), 5, 8)):
            out = oc.experiment(oc.Config(participants_per_round=k, rounds=rounds, seed=seed, max_executors=32), fl,
                                features=8, classes=12, alpha=0.03, train=True, lr=0.05)
            assert np.array_equal(np.array(out["accuracy_series"]), g[f"s{seed}_{name}_acc"])
            assert np.array_equal(out["final_params"], g[f"s{seed}_{name}_params"])
