"""Generate golden fixtures by running the REAL reference (fedsim) in this container.

Usage (build container only -- /root/reference does not exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

The reference is imported read-only from /root/reference/pkg/src.  Outputs:

* flcore.npz          -- fl_core: seeds, dataset, partition, loss/grad,
                         local_train deltas (ragged / reshuffle / empty),
                         fedavg, accuracy.
* orchestration.json  -- fleets, case-study schedules, DES traces + round
                         reports (fuzzed), run_experiment reports.
* round_c10.npz / round_c62.npz -- one FL round at FEMNIST shape
                         (F=784, C=10 / 62, 10 clients x 6400 samples, B=64):
                         participants, final params, accuracy, two deltas.
* headline_rounds.npz -- bench.py's round shape (128-client fleet, budgets
                         10..100, 100 participants, F=784, C=10) at 640
                         samples/client: params after each of 10 rounds
                         (lr 0.1; headline_rounds_lr1e-3.npz: lr 1e-3).
* a8.npz              -- acceptance criterion A8's 30 convergence runs.

These fixtures pin the oracle (tests/test_oracle_golden.py) and the product
(tests/test_gpu_parity.py, tests/test_host_parity.py).
"""

from __future__ import annotations

import json
import os
import random
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _ref():
    sys.dont_write_bytecode = True
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import fedsim  # noqa: F401
    from fedsim import cost_model, engine, fl_core, profiles, scheduler
    return fedsim, cost_model, engine, fl_core, profiles, scheduler


def _jsonable(obj):
    if isinstance(obj, dict):
        return {str(k): _jsonable(v) for k, v in obj.items()}
    if isinstance(obj, (list, tuple)):
        return [_jsonable(v) for v in obj]
    if isinstance(obj, (np.floating,)):
        return float(obj)
    if isinstance(obj, (np.integer,)):
        return int(obj)
    return obj


def report_dict(rep):
    return {
        "round": rep.round_index,
        "makespan": rep.makespan,
        "utilization": rep.utilization,
        "vacancy_area": rep.vacancy_area,
        "throughput": rep.throughput,
        "parallelism_timeline": rep.parallelism_timeline,
        "per_client_times": rep.per_client_times,
        "per_client_start": rep.per_client_start,
        "per_client_end": rep.per_client_end,
        "per_client_budget": rep.per_client_budget,
        "degenerate": rep.degenerate,
    }


def fleet_rows(fleet):
    return [
        [p.client_id, p.resource_budget, p.workload.num_samples, p.workload.batch_size,
         p.workload.model_layers, p.workload.seq_len, p.workload.extra_model_factor,
         [[ph.work_fraction, ph.demand] for ph in p.demand_profile]]
        for p in fleet
    ]


# Fleet-distribution cases shared with the tests (kwargs of DistributionSpec).
FLEET_CASES = [
    dict(n=10, seed=1, spec=dict(budget_levels=[10, 15, 30, 40, 50, 65, 80], num_samples=6400, batch_size=64)),
    dict(n=120, seed=7, spec=dict(budget_levels=[10, 20, 30, 40, 50, 60, 70, 80, 90, 100])),
    dict(n=300, seed=3, spec=dict(budget_levels=[10, 25, 50], budget_weights=[0.5, 0.3, 0.2],
                                  num_samples=[16, 32, 64, 128, 256, 512, 1024], batch_size=[16, 32],
                                  model_layers=[1, 2, 4], seq_len=[64, 128], extra_model_factor=[1.0, 1.5, 2.0],
                                  demand_profiles=["", "0.7:90;0.3:20", "0.5:60;0.5:100"],
                                  demand_weights=[0.5, 0.25, 0.25])),
    dict(n=2800, seed=17, spec=dict(budget_levels=[10, 15, 30, 40, 50, 65, 80])),
]

# DES cases: (fleet case index, participants, FleetConfig kwargs)
DES_CASES = [
    (0, 10, dict()),
    (0, 10, dict(scheduler_kind="greedy")),
    (0, 10, dict(scheduler_kind="greedy", dynamic_parallelism=False)),
    (1, 100, dict(theta=100.0, max_executors=16)),
    (1, 100, dict(theta=150.0, max_executors=16)),
    (1, 60, dict(theta=120.0, max_executors=4, launch_latency=0.5, upload_latency=0.25, terminate_latency=0.1)),
    (2, 80, dict(theta=100.0, max_executors=12)),
    (2, 80, dict(theta=170.0, max_executors=10, scheduler_kind="greedy")),
    (2, 50, dict(theta=100.0, max_executors=3, dynamic_parallelism=False, launch_latency=1.0)),
    (3, 200, dict(theta=100.0, max_executors=10, seed=17)),
]

# run_experiment without training: (fleet case, FleetConfig kwargs)
EXP_CASES = [
    (1, dict(participants_per_round=20, rounds=3, seed=9, max_executors=8)),
    (2, dict(participants_per_round=30, rounds=2, seed=4, theta=150.0, max_executors=16)),
    (3, dict(participants_per_round=100, rounds=2, seed=17, max_executors=10)),
]

# run_experiment with training (small model): (fleet kwargs, FleetConfig kwargs, DataParams kwargs, lr)
TRAIN_CASES = [
    (dict(n=8, seed=2, spec=dict(budget_levels=[10, 30, 50], num_samples=[100, 150, 200], batch_size=[32, 50])),
     dict(participants_per_round=5, rounds=3, seed=3, max_executors=8),
     dict(features=4, classes=4, alpha=0.5), 0.1),
    (dict(n=6, seed=5, spec=dict(budget_levels=[25, 50], num_samples=[64, 96, 100], batch_size=[16, 30])),
     dict(participants_per_round=6, rounds=2, seed=5, aggregation="async", async_buffer=4),
     dict(features=6, classes=5, alpha=0.3), 0.2),
    (dict(n=12, seed=11, spec=dict(budget_levels=[10, 15, 30, 40, 50, 65, 80], num_samples=[128, 200, 333], batch_size=[32, 64])),
     dict(participants_per_round=8, rounds=2, seed=11, aggregation="async", async_buffer=3, theta=150.0),
     dict(features=16, classes=10, alpha=0.5), 0.05),
]


def gen_flcore(fl_core, profiles):
    out = {}
    seeds = [fl_core.stable_seed(*p) for p in [("train", 1, 0, "c0000"), ("data", 1), ("partition", 1),
                                                ("local_train", 123), ("x",), ("train", 9, 3, "A")]]
    out["seeds"] = np.array(seeds, dtype=np.uint64)
    tr, te = fl_core.make_synthetic_dataset(5, 3, 200, seed=42)
    out["ds_train_x"], out["ds_train_y"] = tr.features, tr.labels
    out["ds_test_x"], out["ds_test_y"] = te.features, te.labels
    tr, _ = fl_core.make_synthetic_dataset(3, 4, 2000, seed=5)
    clients = [(f"k{i}", n) for i, n in enumerate([100, 250, 17, 0, 400])]
    shards = fl_core.partition_noniid(tr, clients, 0.3, seed=11)
    for cid, _ in clients:
        out[f"part_{cid}_y"] = shards[cid].labels
        out[f"part_{cid}_x"] = shards[cid].features
    rng = np.random.default_rng(0)
    x = rng.standard_normal((20, 3))
    y = rng.integers(0, 4, size=20)
    p = rng.standard_normal(16) * 0.5
    loss, grad = fl_core.loss_and_grad(p, x, y, 4)
    out["lg_x"], out["lg_y"], out["lg_p"] = x, y, p
    out["lg_loss"], out["lg_grad"] = np.array(loss), grad
    # local_train cases: (F, C, n_rows, num_samples, batch, lr, seed)
    lt_cases = [(2, 4, 200, 200, 32, 0.1, 5), (4, 3, 100, 500, 64, 0.5, 1), (6, 5, 77, 77, 10, 0.2, "s"),
                (3, 4, 50, 130, 64, 0.3, 99), (8, 10, 300, 320, 64, 0.1, 7), (2, 4, 0, 100, 32, 0.1, 0)]
    out["lt_cases"] = np.array([[F, C, n, ns, b, lr] for F, C, n, ns, b, lr, _ in lt_cases])
    for i, (F, C, n, ns, b, lr, sd) in enumerate(lt_cases):
        trn, _ = fl_core.make_synthetic_dataset(F, C, max(n * 2, 10), seed=100 + i)
        shard = fl_core.DatasetShard("a", trn.features[:n], trn.labels[:n])
        params = rng.standard_normal(F * C + C) * 0.1
        wl = profiles.WorkloadSpec(num_samples=ns, batch_size=b)
        d = fl_core.local_train(params, shard, wl, lr, C, seed=sd)
        out[f"lt{i}_x"], out[f"lt{i}_y"], out[f"lt{i}_p"], out[f"lt{i}_d"] = shard.features, shard.labels, params, d
    out["lt_seeds"] = np.array([str(c[-1]) for c in lt_cases])
    # fedavg goldens
    base = rng.standard_normal(33)
    ds = [rng.standard_normal(33) for _ in range(7)]
    ws = [float(v) for v in rng.integers(1, 1024, size=7)]
    out["fa_base"], out["fa_deltas"], out["fa_w"] = base, np.stack(ds), np.array(ws)
    out["fa_out"] = fl_core.fedavg(ds, ws, base)
    # accuracy
    trn, tst = fl_core.make_synthetic_dataset(7, 6, 500, seed=8)
    pa = rng.standard_normal(7 * 6 + 6)
    out["acc_p"], out["acc_x"], out["acc_y"] = pa, tst.features, tst.labels
    out["acc"] = np.array(fl_core.evaluate_accuracy(pa, tst))
    np.savez_compressed(os.path.join(HERE, "flcore.npz"), **out)


def gen_orchestration(fedsim, cost_model, engine, profiles, scheduler):
    from collections import deque
    doc = {"fleets": [], "des": [], "experiments": [], "selection": [], "maxmin": [], "work": []}
    fleets = []
    for case in FLEET_CASES:
        f = profiles.generate_fleet(profiles.DistributionSpec(**case["spec"]), case["n"], case["seed"])
        fleets.append(f)
        doc["fleets"].append({"case": case, "rows": fleet_rows(f)})
    # scheduler case study
    pend = [scheduler.Participant(chr(65 + i), float(b)) for i, b in enumerate(profiles.CASE_STUDY_BUDGETS)]
    st = scheduler.SchedulerState([], 0, deque(range(8)))
    ra = scheduler.schedule_resource_aware(st, list(pend), 8, 100.0)
    st = scheduler.SchedulerState([], 0, deque(range(8)))
    gr = scheduler.schedule_greedy(st, list(pend), 8, 100.0)
    doc["case_study"] = {"ra": [[e.client_id, e.resource_budget, e.executor_id] for e in ra],
                         "greedy": [[e.client_id, e.resource_budget, e.executor_id] for e in gr]}
    # random scheduler calls
    rnd = random.Random(1234)
    sched_calls = []
    for _ in range(200):
        n = rnd.randint(0, 12)
        pend = [scheduler.Participant(f"p{rnd.randint(0, 99):02d}", float(rnd.choice([5, 10, 15, 25, 40, 50, 65, 80, 100])))
                for _ in range(n)]
        running = [float(rnd.choice([10, 20, 30])) for _ in range(rnd.randint(0, 3))]
        ex = rnd.randint(0, 6)
        planned = rnd.randint(0, 3)
        target = rnd.randint(0, 12)
        theta = rnd.choice([60.0, 100.0, 150.0])
        kind = rnd.choice(["resource-aware", "greedy"])
        st = scheduler.SchedulerState(list(running), planned, deque(range(ex)))
        got = scheduler.SCHEDULERS[kind](st, list(pend), target, theta)
        sched_calls.append({"kind": kind, "pending": [[p.client_id, p.resource_budget] for p in pend],
                            "running": running, "executors": ex, "planned": planned, "target": target,
                            "theta": theta, "out": [[e.client_id, e.resource_budget, e.executor_id] for e in got],
                            "state_after": [st.running_budgets, st.planned_count, list(st.available_executors)]})
    doc["sched_calls"] = sched_calls
    # water-filling
    for _ in range(300):
        n = rnd.randint(0, 9)
        caps = [float(rnd.choice([5, 10, 12.5, 20, 33.3, 50, 65, 80, 100])) for _ in range(n)]
        dem = [float(rnd.choice([10, 20, 40, 60, 90, 100])) for _ in range(n)]
        doc["maxmin"].append([caps, dem, cost_model.maxmin_allocate(caps, dem)])
    for f in fleets[2][:50]:
        w = f.workload
        doc["work"].append([[w.num_samples, w.batch_size, w.model_layers, w.seq_len, w.extra_model_factor],
                            cost_model.work_units(w, cost_model.CostCoefficients())])
    # DES
    for fi, n, kw in DES_CASES:
        fleet = {p.client_id: p for p in fleets[fi]}
        ids = sorted(fleet)
        part = random.Random(f"des:{fi}:{n}:{sorted(kw.items())}").sample(ids, n)
        cfg = profiles.FleetConfig(**kw)
        rep, seg = engine.run_round(fleet, part, cfg, t0=0.0, round_index=0)
        doc["des"].append({"fleet": fi, "participants": part, "cfg": kw, "report": report_dict(rep), "trace": seg})
    # selection streams
    for seed in (1, 2, 9, 17):
        r = random.Random(f"{seed}:selection")
        ids = [f"c{i:04d}" for i in range(120)]
        doc["selection"].append({"seed": seed, "picks": [r.sample(ids, 10) for _ in range(5)]})
    # run_experiment without training
    for fi, kw in EXP_CASES:
        cfg = profiles.FleetConfig(**kw)
        trace = []
        rep = engine.run_experiment(cfg, fleets[fi], trace=trace)
        doc["experiments"].append({"fleet": fi, "cfg": kw, "participants": rep.participants,
                                   "rounds": [report_dict(r) for r in rep.rounds],
                                   "total_time": rep.total_time, "trace_len": len(trace),
                                   "trace_tail": trace[-40:]})
    with open(os.path.join(HERE, "orchestration.json"), "w") as fh:
        json.dump(_jsonable(doc), fh, sort_keys=True)


def gen_train_experiments(engine, profiles):
    out = {}
    meta = []
    for i, (fk, ck, dk, lr) in enumerate(TRAIN_CASES):
        fleet = profiles.generate_fleet(profiles.DistributionSpec(**fk["spec"]), fk["n"], fk["seed"])
        rep = engine.run_experiment(profiles.FleetConfig(**ck), fleet, engine.DataParams(**dk),
                                    engine.TrainParams(enabled=True, lr=lr))
        out[f"tr{i}_params"] = rep.final_params
        out[f"tr{i}_acc"] = np.array(rep.accuracy_series)
        meta.append({"fleet": fk, "cfg": ck, "data": dk, "lr": lr, "participants": rep.participants})
    out["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(os.path.join(HERE, "train_small.npz"), **out)


def gen_round(engine, profiles, fl_core, classes):
    fleet = profiles.generate_fleet(
        profiles.DistributionSpec(budget_levels=(10, 15, 30, 40, 50, 65, 80), num_samples=6400, batch_size=64), 10, 1)
    cfg = profiles.FleetConfig(participants_per_round=10, rounds=1, seed=1, theta=100.0)
    rep = engine.run_experiment(cfg, fleet, engine.DataParams(features=784, classes=classes, alpha=0.5),
                                engine.TrainParams(enabled=True, lr=0.1))
    np.savez_compressed(
        os.path.join(HERE, f"round_c{classes}.npz"),
        participants=np.array(rep.participants[0]),
        params=rep.final_params,
        acc=np.array(rep.accuracy_series),
        makespan=np.array(rep.rounds[0].makespan),
    )


HEADLINE = dict(n=128, seed=1, budgets=tuple(range(10, 101, 10)), num_samples=640, batch=64, participants=100,
                theta=100.0, max_executors=18, rounds=10, features=784, classes=10, lr=0.1)


def gen_headline(engine, profiles, fl_core, lr=None, name="headline_rounds.npz"):
    """bench.py's round shape (128-client fleet, budgets 10..100, 100 participants/round, theta 100, 18
    executors, F=784, C=10) at 640 samples per client, 10 rounds.  The params after EVERY round are
    captured from the reference's own evaluate_accuracy call (engine.py:352 passes the new params).

    At bench.py's lr = 0.1 the reference's fp64 softmax saturates to an exact one-hot after round 1 (the
    784-feature Gaussian classes are far apart), so every later delta is exactly 0 and the params stop
    moving; lr = 1e-3 (headline_rounds_lr1e-3.npz) keeps the gradients alive for all 10 rounds."""
    h = dict(HEADLINE)
    if lr is not None:
        h["lr"] = lr
    fleet = profiles.generate_fleet(profiles.DistributionSpec(budget_levels=h["budgets"], num_samples=h["num_samples"],
                                                              batch_size=h["batch"]), h["n"], h["seed"])
    cfg = profiles.FleetConfig(participants_per_round=h["participants"], rounds=h["rounds"], seed=h["seed"],
                               theta=h["theta"], max_executors=h["max_executors"])
    snaps = []
    orig = fl_core.evaluate_accuracy

    def spy(params, dataset):
        snaps.append(np.array(params, copy=True))
        return orig(params, dataset)

    fl_core.evaluate_accuracy = spy
    try:
        rep = engine.run_experiment(cfg, fleet, engine.DataParams(features=h["features"], classes=h["classes"],
                                                                   alpha=0.5),
                                    engine.TrainParams(enabled=True, lr=h["lr"]))
    finally:
        fl_core.evaluate_accuracy = orig
    assert len(snaps) == h["rounds"]
    np.savez_compressed(os.path.join(HERE, name), params=np.stack(snaps).astype(np.float64),
                        acc=np.array(rep.accuracy_series), participants=np.array(rep.participants),
                        makespans=np.array([r.makespan for r in rep.rounds]), meta=np.array(json.dumps(h)))


def gen_a8(engine, profiles):
    """The reference's acceptance criterion A8 (pkg/tests/test_acceptance.py:300-336): the accuracy series
    of all 30 convergence runs (5 seeds x 3 comparisons x 2 arms)."""
    from fedsim.profiles import ClientProfile, WorkloadSpec

    def fleet_of(n, budgets, factor=1.0, samples=100):
        return [ClientProfile(f"c{i:02d}", budgets[i % len(budgets)],
                              WorkloadSpec(num_samples=samples, batch_size=50, extra_model_factor=factor))
                for i in range(n)]

    def run(fleet, k, rounds, seed):
        cfg = profiles.FleetConfig(participants_per_round=k, rounds=rounds, seed=seed, max_executors=32)
        return engine.run_experiment(cfg, fleet, engine.DataParams(features=8, classes=12, alpha=0.03),
                                     engine.TrainParams(enabled=True, lr=0.05))

    out = {}
    for seed in range(5):
        arms = {
            "wide": run(fleet_of(40, [10]), 20, 6, seed), "narrow": run(fleet_of(40, [10]), 5, 12, seed),
            "light": run(fleet_of(20, [50]), 10, 8, seed), "heavy": run(fleet_of(20, [50], factor=2.0), 10, 8, seed),
            "uniform": run(fleet_of(20, [100]), 5, 8, seed),
            "hetero": run(fleet_of(20, [10, 15, 30, 50, 80]), 5, 8, seed),
        }
        for name, rep in arms.items():
            out[f"s{seed}_{name}_acc"] = np.array(rep.accuracy_series)
            out[f"s{seed}_{name}_params"] = rep.final_params
            out[f"s{seed}_{name}_total"] = np.array(rep.total_time)
    np.savez_compressed(os.path.join(HERE, "a8.npz"), **out)


def gen_outputs(engine, profiles):
    """Reference `simulate` writers (cli.py:38-87) on one untrained experiment."""
    from pathlib import Path

    from fedsim import cli, metrics
    out = Path(HERE) / "outputs"
    out.mkdir(exist_ok=True)
    case = FLEET_CASES[2]
    fleet = profiles.generate_fleet(profiles.DistributionSpec(**case["spec"]), case["n"], case["seed"])
    cfg = profiles.FleetConfig(participants_per_round=12, rounds=2, seed=4, theta=120.0, max_executors=6)
    trace = []
    rep = engine.run_experiment(cfg, fleet, trace=trace)
    metrics.write_trace_jsonl(trace, out / "trace.jsonl")
    cli._write_rounds_csv(out / "rounds.csv", rep)
    cli._write_clients_csv(out / "clients.csv", rep)
    profiles.save_fleet(fleet, out / "fleet.csv")


def main():
    fedsim, cost_model, engine, fl_core, profiles, scheduler = _ref()
    gen_outputs(engine, profiles)
    gen_flcore(fl_core, profiles)
    gen_orchestration(fedsim, cost_model, engine, profiles, scheduler)
    gen_train_experiments(engine, profiles)
    for c in (10, 62):
        gen_round(engine, profiles, fl_core, c)
    gen_headline(engine, profiles, fl_core)
    gen_headline(engine, profiles, fl_core, lr=1e-3, name="headline_rounds_lr1e-3.npz")
    gen_a8(engine, profiles)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
