"""Product host logic vs the reference goldens (CPU only): fleets, cost model,
schedulers, executor manager, the native DES (bit-exact traces and reports),
run_experiment without training, datasets, partitions and batch order."""

import json
import os
import random
from collections import deque

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import flmath as fm
from oracle import orchestration as oc

import paper_2305_15668_b200 as fh
from paper_2305_15668_b200 import planner, roundsim, spec, training
from paper_2305_15668_b200.errors import ConfigError

with open(os.path.join(GOLDEN, "orchestration.json")) as fh_:
    ORCH = json.load(fh_)
FL = np.load(os.path.join(GOLDEN, "flcore.npz"))


def _mg():
    import importlib.util
    sp = importlib.util.spec_from_file_location("mg", os.path.join(GOLDEN, "make_golden.py"))
    m = importlib.util.module_from_spec(sp)
    sp.loader.exec_module(m)
    return m


MG = _mg()


def product_fleet(case):
    return fh.generate_fleet(fh.DistributionSpec(**case["spec"]), case["n"], case["seed"])


def rows(fleet):
    return [[p.client_id, p.resource_budget, p.workload.num_samples, p.workload.batch_size, p.workload.model_layers,
             p.workload.seq_len, p.workload.extra_model_factor,
             [[ph.work_fraction, ph.demand] for ph in p.demand_profile]] for p in fleet]


def norm(x):
    return json.loads(json.dumps(x, sort_keys=True))


def report_dict(rep):
    return {"round": rep.round_index, "makespan": rep.makespan, "utilization": rep.utilization,
            "vacancy_area": rep.vacancy_area, "throughput": rep.throughput,
            "parallelism_timeline": rep.parallelism_timeline, "per_client_times": rep.per_client_times,
            "per_client_start": rep.per_client_start, "per_client_end": rep.per_client_end,
            "per_client_budget": rep.per_client_budget, "degenerate": rep.degenerate}


def test_fleets_bit_exact():
    for case, want in zip(MG.FLEET_CASES, ORCH["fleets"]):
        assert rows(product_fleet(case)) == want["rows"]


def test_fleet_csv_roundtrip(tmp_path):
    f = product_fleet(MG.FLEET_CASES[2])
    path = tmp_path / "fleet.csv"
    fh.save_fleet(f, path)
    assert fh.load_fleet(path) == f


def test_fleet_validation():
    with pytest.raises(ConfigError):
        fh.WorkloadSpec(batch_size=0)
    with pytest.raises(ConfigError):
        fh.ClientProfile("a", 101)
    with pytest.raises(ConfigError):
        fh.DistributionSpec(budget_levels=()).validate()
    with pytest.raises(ConfigError, match="exceeds"):
        fh.FleetConfig(participants_per_round=3).validate(fleet_size=2)


def test_work_units_and_maxmin():
    for caps, dem, want in ORCH["maxmin"]:
        assert fh.maxmin_allocate(caps, dem) == want
    for (ns, b, l, s, x), want in ORCH["work"]:
        assert fh.work_units(fh.WorkloadSpec(ns, b, l, s, x), fh.CostCoefficients()) == want


def test_scheduler_api_calls():
    for c in ORCH["sched_calls"]:
        st = fh.SchedulerState(list(c["running"]), c["planned"], deque(range(c["executors"])))
        pend = [fh.Participant(cid, b) for cid, b in c["pending"]]
        got = planner.SCHEDULERS[c["kind"]](st, pend, c["target"], c["theta"])
        assert [[e.client_id, e.resource_budget, e.executor_id] for e in got] == c["out"]
        assert [st.running_budgets, st.planned_count, list(st.available_executors)] == c["state_after"]


def test_executor_manager_case_study():
    parts = [fh.Participant(p.client_id, p.resource_budget) for p in fh.case_study_fleet()]
    mgr = planner.ExecutorManager(8, "resource-aware", 100.0)
    mgr.begin_round(parts)
    launches = mgr.kickoff(0.0)
    assert [e.client_id for e, _ in launches] == ["A", "D", "H"]
    d = next(e for e, _ in launches if e.client_id == "D")
    for kind in (planner.RequestKind.REGISTER, planner.RequestKind.TRAINING_COMPLETE,
                 planner.RequestKind.MODEL_UPLOADED):
        mgr.on_request(planner.ClientRequest("D", kind), 5.0)
    assert [e.client_id for e, _ in mgr.on_slot_freed(d.executor_id, 5.0)] == ["B", "E"]
    assert mgr.occupied_budget() == 100.0
    fixed = planner.ExecutorManager(8, "greedy", 100.0, dynamic_parallelism=False)
    fixed.begin_round(parts)
    assert [e.client_id for e, _ in fixed.kickoff(0.0)] == ["A", "B", "C"]


def _des_entry(entry):
    fleets = [product_fleet(c) for c in MG.FLEET_CASES]
    fleet = {p.client_id: p for p in fleets[entry["fleet"]]}
    return fh.run_round(fleet, entry["participants"], fh.FleetConfig(**entry["cfg"]))


@pytest.mark.parametrize("i", range(len(MG.DES_CASES)))
def test_native_des_bit_exact(i):
    entry = ORCH["des"][i]
    rep, seg = _des_entry(entry)
    assert norm(seg) == entry["trace"]
    assert norm(report_dict(rep)) == entry["report"]


def test_native_des_random_vs_oracle():
    """Fuzz the native DES against the oracle restatement (phases, latencies, both policies)."""
    rnd = random.Random(3)
    for trial in range(40):
        n = rnd.randint(1, 40)
        dist = dict(budget_levels=rnd.sample([5, 10, 15, 20, 30, 40, 50, 65, 80, 100], rnd.randint(1, 5)),
                    num_samples=[rnd.choice([0, 16, 64, 500, 1000]) for _ in range(2)],
                    batch_size=[16, 32], model_layers=[1, 3], seq_len=[32, 128],
                    extra_model_factor=[1.0, 2.5],
                    demand_profiles=["", "0.7:90;0.3:20", "0.2:10;0.5:100;0.3:35"])
        pf = fh.generate_fleet(fh.DistributionSpec(**dist), n, trial)
        of = oc.fleet(n, trial, **dist)
        cfg = dict(theta=rnd.choice([100.0, 120.0, 150.0, 300.0]), max_executors=rnd.randint(1, 12),
                   scheduler_kind=rnd.choice(["resource-aware", "greedy"]),
                   dynamic_parallelism=rnd.random() < 0.7,
                   launch_latency=rnd.choice([0.0, 0.5]), upload_latency=rnd.choice([0.0, 0.25]),
                   terminate_latency=rnd.choice([0.0, 0.1]))
        ids = sorted(p.client_id for p in pf)
        part = rnd.sample(ids, rnd.randint(1, n))
        t0 = rnd.choice([0.0, 17.25])
        rep, seg = fh.run_round({p.client_id: p for p in pf}, part, fh.FleetConfig(**cfg), t0=t0, round_index=trial)
        orep, oseg = oc.simulate_round({c.client_id: c for c in of}, part, oc.Config(**cfg), t0=t0,
                                       round_index=trial)
        assert norm(seg) == norm(oseg)
        assert norm(report_dict(rep)) == norm(orep)


def test_des_errors():
    fleet = {p.client_id: p for p in fh.case_study_fleet()}
    with pytest.raises(ConfigError, match="not in fleet"):
        fh.run_round(fleet, ["nope"], fh.FleetConfig())
    with pytest.raises(ConfigError, match="theta"):
        fh.run_round(fleet, ["D"], fh.FleetConfig(theta=60.0))


def test_empty_round():
    rep, seg = fh.run_round({}, [], fh.FleetConfig())
    orep, oseg = oc.simulate_round({}, [], oc.Config())
    assert norm(seg) == norm(oseg) and rep.degenerate


def test_trace_metrics_match_native_report():
    entry = ORCH["des"][4]
    rep, seg = _des_entry(entry)
    again = roundsim.build_round_report(seg)
    assert norm(report_dict(again)) == norm(report_dict(rep))


def test_experiments_without_training():
    fleets = [product_fleet(c) for c in MG.FLEET_CASES]
    for entry in ORCH["experiments"]:
        trace = []
        rep = fh.run_experiment(fh.FleetConfig(**entry["cfg"]), fleets[entry["fleet"]], trace=trace)
        assert rep.participants == entry["participants"]
        assert norm([report_dict(r) for r in rep.rounds]) == entry["rounds"]
        assert rep.total_time == entry["total_time"]
        assert len(trace) == entry["trace_len"] and norm(trace[-40:]) == entry["trace_tail"]


def test_dataset_partition_and_batch_order():
    tr, te = training.make_synthetic_dataset(5, 3, 200, seed=42)
    assert np.array_equal(tr.features, FL["ds_train_x"]) and np.array_equal(te.labels, FL["ds_test_y"])
    tr, _ = training.make_synthetic_dataset(3, 4, 2000, seed=5)
    clients = [(f"k{i}", n) for i, n in enumerate([100, 250, 17, 0, 400])]
    shards = training.partition_noniid(tr, clients, 0.3, seed=11)
    for cid, _ in clients:
        assert np.array_equal(shards[cid].labels, FL[f"part_{cid}_y"])
        assert np.array_equal(shards[cid].features, FL[f"part_{cid}_x"])
    for n, ns, b, seed in [(200, 200, 32, 5), (100, 500, 64, 1), (77, 77, 10, "s"), (50, 130, 64, 99), (0, 10, 4, 0),
                           (6400, 6400, 64, 123456), (33, 0, 8, 1)]:
        plan = fm.batch_plan(n, ns, b, seed)
        perm = training.batch_permutations(n, ns, b, seed)
        bpe = -(-n // b) if n else 1
        for s, rows_ in enumerate(plan):
            e, j = divmod(s, bpe)
            assert np.array_equal(perm[e * n + j * b: e * n + j * b + len(rows_)], rows_)
    assert training.stable_seed("train", 1, 0, "c0000") == int(FL["seeds"][0])


def test_native_round_seeds_match_stable_seed():
    import ctypes as C
    from paper_2305_15668_b200 import _abi
    ids = [f"c{i:04d}" for i in range(50)] + ["it's", 'q"x', "ü-id", "a\\b", ""]
    arr = (C.c_char_p * len(ids))(*[repr(c).encode() for c in ids])
    ts = np.zeros(len(ids), np.uint64)
    rs = np.zeros(len(ids), np.uint64)
    for seed, r in [(1, 0), (17, 5), (-3, 2), (2 ** 40, 123)]:
        _abi.check(_abi.lib.fedhc_round_seeds(seed, r, arr, len(ids), ts.ctypes.data, rs.ctypes.data))
        for i, c in enumerate(ids):
            t = fm.seed_of("train", seed, r, c)
            assert int(ts[i]) == t and int(rs[i]) == fm.seed_of("local_train", t)


def test_native_permutations_match_numpy():
    seeds = [5, 99, 123456, 4294967295, 0, 31337]
    rows = [6400, 1, 77, 1000, 2, 300]
    perms = [1, 3, 2, 1, 4, 2]
    out = training.native_permutations(seeds, rows, perms)
    at = 0
    for s, n, k in zip(seeds, rows, perms):
        g = np.random.default_rng(s)
        want = np.concatenate([g.permutation(n) for _ in range(k)])
        assert np.array_equal(out[at:at + n * k], want)
        at += n * k


def test_output_files_byte_identical(tmp_path):
    """trace.jsonl / rounds.csv / clients.csv / fleet.csv vs the reference's own writers (cli.py:38-87)."""
    from paper_2305_15668_b200 import reports
    case = MG.FLEET_CASES[2]
    fleet = product_fleet(case)
    cfg = fh.FleetConfig(participants_per_round=12, rounds=2, seed=4, theta=120.0, max_executors=6)
    trace = []
    rep = fh.run_experiment(cfg, fleet, trace=trace)
    reports.write_outputs(str(tmp_path), rep, trace=trace, fleet=fleet, config=cfg)
    for name in ("trace.jsonl", "rounds.csv", "clients.csv", "fleet.csv"):
        want = open(os.path.join(GOLDEN, "outputs", name), "rb").read()
        assert open(tmp_path / name, "rb").read() == want, name
    summary = json.load(open(tmp_path / "summary.json"))
    assert summary["participants"] == rep.participants and summary["total_time"] == rep.total_time


def test_dirichlet_counts_quotas():
    from paper_2305_15668_b200.devicedata import dirichlet_counts
    sizes = [0, 1, 17, 640, 6400, 1024]
    c = dirichlet_counts(sizes, 10, 0.5, seed=3)
    assert c.shape == (6, 10) and (c >= 0).all()
    assert list(c.sum(axis=1)) == sizes
    flat = dirichlet_counts([2000] * 20, 4, 1000.0, seed=1)
    assert np.all(np.abs(flat / 2000 - 0.25) < 0.05)            # alpha -> inf: near IID
    skew = dirichlet_counts([500] * 30, 4, 0.05, seed=1)
    assert np.mean(skew.max(axis=1) / 500) > 0.7                 # alpha -> 0: concentrated


def test_lean_round_report_matches_full_run():
    """RoundSimulator.run_lean (the serving planner's DES call: reused buffers, per-client dicts on demand)
    produces exactly RoundSimulator.run's report."""
    import numpy as np
    import paper_2305_15668_b200 as fh
    from paper_2305_15668_b200.roundsim import RoundSimulator
    fleet = fh.generate_fleet(fh.DistributionSpec(budget_levels=(10, 30, 50, 80)), 40, 5)
    by_id = {p.client_id: p for p in fleet}
    cfg = fh.FleetConfig(theta=100.0, max_executors=6, participants_per_round=12, seed=3)
    sim = RoundSimulator(by_id)
    rng = np.random.default_rng(1)
    for r in range(4):
        who = [sim.ids[i] for i in rng.choice(len(sim.ids), 12, replace=False)]
        full, _ = sim.run(who, cfg, t0=1.5 * r, round_index=r, want_trace=False)
        lean = sim.run_lean(np.array([sim.index[c] for c in who], np.int32), who, cfg, t0=1.5 * r, round_index=r)
        assert lean.makespan == full.makespan
        assert lean.full() == full
        assert lean.per_client_times == full.per_client_times  # attribute access materialises


@pytest.mark.parametrize("alpha,seed", [(0.05, 3), (0.3, 7), (5.0, 1)])
def test_partition_rows_vs_oracle_shortfall(alpha, seed):
    """training.partition_rows (ndarray pools, the device dataset's partition) == the oracle's list-pool
    restatement of fl_core.py:62-115, including the richest-pool shortfall path (a dataset that the clients
    nearly exhaust, so late clients run out of their Dirichlet classes) and empty clients."""
    tr, _ = training.make_synthetic_dataset(3, 7, 1500, seed=seed)
    n_train = len(tr.labels)
    sizes = [37, 0, 150, 1, 90, 200, 64, 128, 0, 300]
    sizes.append(n_train - sum(sizes) - 3)  # all but 3 rows taken: the tail clients hit empty class pools
    clients = [(f"p{i}", n) for i, n in enumerate(sizes)]
    got = training.partition_rows(tr.labels, 7, clients, alpha, seed + 100)
    want = fm.dirichlet_partition(fm.Data(tr.features, tr.labels, 7), clients, alpha, seed + 100)
    for cid, n in clients:
        assert len(got[cid]) == n
        assert np.array_equal(tr.labels[got[cid]], want[cid].labels)
        assert np.array_equal(tr.features[got[cid]], want[cid].features)
