"""Oracle restatement of the reference control plane (TEST INFRASTRUCTURE ONLY).

Restates, with the same fp64 operation order and tie-breaks, the parts of the
reference that decide *which* clients run *when* and with which sample counts:

* fleet generation        -- profiles.py:19-205
* cost model              -- cost_model.py:18-102
* double-pointer / greedy -- scheduler.py:30-130
* executor manager        -- executor_manager.py:71-238
* round DES               -- engine.py:53-230
* round metrics           -- metrics.py:21-167
* experiment loop         -- engine.py:279-368 (selection, training, sync/async FedAvg)

Plain dicts and small classes are used instead of the reference's dataclasses;
the observable outputs (schedules, traces, reports, params) are what the tests
compare.
"""

from __future__ import annotations

import heapq
import math
import random
from collections import deque
from dataclasses import dataclass, field

from . import flmath


class ConfigError(Exception):
    """Mirrors fedsim.errors.ConfigError."""


CAPACITY = 100.0
RANK = {  # metrics.py:21-28
    "ClientLaunched": 0,
    "PhaseCompleted": 1,
    "ClientTrainingComplete": 2,
    "ModelUploaded": 3,
    "SlotFreed": 4,
    "RoundComplete": 5,
}
TIMER_RANK = {"start": 0, "upload_done": 3, "slot_freed": 4}  # engine.py:31-35


# -- fleet (profiles.py) -----------------------------------------------------


@dataclass(frozen=True)
class Workload:
    num_samples: int = 6400
    batch_size: int = 64
    model_layers: int = 2
    seq_len: int = 128
    extra_model_factor: float = 1.0


@dataclass(frozen=True)
class Client:
    client_id: str
    resource_budget: int
    workload: Workload = field(default_factory=Workload)
    phases: tuple = ((1.0, 100.0),)  # (work_fraction, demand)


def parse_phases(text: str) -> tuple:
    """profiles.py:156-168 ('frac:demand;...', empty -> one full-demand phase)."""
    text = text.strip()
    if not text:
        return ((1.0, 100.0),)
    out = []
    for part in text.split(";"):
        a, _, b = part.partition(":")
        out.append((float(a), float(b)))
    return tuple(out)


def fleet(n: int, seed: int, budget_levels=(25, 50, 75, 100), budget_weights=None,
          num_samples=6400, batch_size=64, model_layers=2, seq_len=128,
          extra_model_factor=1.0, demand_profiles=("",), demand_weights=None) -> list[Client]:
    """profiles.py:177-205: one random.Random stream, draws in field order."""
    r = random.Random(f"fleet:{seed}")
    as_list = lambda v: list(v) if isinstance(v, (list, tuple)) else [v]
    digits = max(4, len(str(max(n - 1, 0))))
    out = []
    for i in range(n):
        budget = r.choices(list(budget_levels), weights=budget_weights)[0]
        wl = Workload(
            r.choice(as_list(num_samples)),
            r.choice(as_list(batch_size)),
            r.choice(as_list(model_layers)),
            r.choice(as_list(seq_len)),
            r.choice(as_list(extra_model_factor)),
        )
        demand = r.choices(list(demand_profiles), weights=demand_weights)[0]
        out.append(Client(f"c{i:0{digits}d}", int(budget), wl, parse_phases(demand)))
    return out


CASE_STUDY = (10, 15, 30, 80, 65, 40, 50, 10)  # profiles.py:209


def case_study(workload: Workload | None = None) -> list[Client]:
    """profiles.py:212-218: clients A..H."""
    workload = workload or Workload()
    return [Client(chr(65 + i), b, workload) for i, b in enumerate(CASE_STUDY)]


# -- cost model (cost_model.py) -------------------------------------------


def work_of(w: Workload, alpha: float, beta: float) -> float:
    """cost_model.py:33-45 (same association order)."""
    per_batch = alpha * w.model_layers * w.seq_len * w.batch_size + beta * w.model_layers
    return math.ceil(w.num_samples / w.batch_size) * per_batch * w.extra_model_factor


def water_fill(caps, demands, capacity=CAPACITY):
    """cost_model.py:48-87: capped max-min fair shares by progressive filling."""
    if len(caps) != len(demands):
        raise ConfigError("caps and demands must have equal length")
    for c, d in zip(caps, demands):
        if not 0 < c <= 100:
            raise ConfigError(f"cap {c} outside (0,100]")
        if not 0 < d <= 100:
            raise ConfigError(f"demand {d} outside (0,100]")
    lim = [min(c, d) for c, d in zip(caps, demands)]
    share = [0.0] * len(lim)
    live = list(range(len(lim)))
    left = capacity
    level = 0.0
    while live and left > 1e-12:
        room = min(lim[i] - level for i in live)
        even = left / len(live)
        if room <= even:
            level += room
            left -= room * len(live)
            for i in live:
                share[i] = min(lim[i], level)
            live = [i for i in live if lim[i] - level > 1e-12]
        else:
            level += even
            for i in live:
                share[i] = level
            left = 0.0
    return share


def solo_time(budget, phases, total_work):
    """cost_model.py:97-102."""
    return sum(frac * total_work / (min(budget, dem) / CAPACITY) for frac, dem in phases)


# -- schedulers (scheduler.py) ---------------------------------------------


class SchedState:
    """scheduler.py:30-37."""

    def __init__(self, running=(), planned=0, executors=()):
        self.running = list(running)
        self.planned = planned
        self.free = deque(executors)

    def total(self) -> float:
        return sum(self.running)


def _admit(st: SchedState, cid: str, budget: float, theta: float):
    """scheduler.py:40-52."""
    if budget + st.total() <= theta + 1e-9 and st.free:
        ex = st.free.popleft()
        st.running.append(budget)
        st.planned += 1
        return (cid, budget, ex)
    return None


def pick_resource_aware(st: SchedState, pending, n_target: int, theta: float):
    """scheduler.py:55-98: alternate smallest / largest budget."""
    srt = sorted(pending, key=lambda p: (p[1], p[0]))
    lo, hi = 0, len(srt) - 1
    use_hi = True
    got = []
    ok = lambda: st.planned < n_target and st.total() < theta - 1e-9
    while ok() and lo <= hi:
        e = _admit(st, srt[lo][0], srt[lo][1], theta)
        if e is None:
            return got
        got.append(e)
        lo += 1
        if not ok():
            return got
        if lo > hi:
            break
        if use_hi:
            e = _admit(st, srt[hi][0], srt[hi][1], theta)
            if e is None:
                use_hi = False
            else:
                got.append(e)
                hi -= 1
    return got


def pick_greedy(st: SchedState, pending, n_target: int, theta: float):
    """scheduler.py:101-124: FIFO with head-of-line blocking."""
    got = []
    for cid, b in pending:
        if not (st.planned < n_target and st.total() < theta - 1e-9):
            break
        e = _admit(st, cid, b, theta)
        if e is None:
            break
        got.append(e)
    return got


POLICIES = {"resource-aware": pick_resource_aware, "greedy": pick_greedy}


# -- executor manager (executor_manager.py) ---------------------------------


class Manager:
    """executor_manager.py:81-238 (slots, record table, status monitor)."""

    def __init__(self, n_exec, policy, theta, dynamic=True, emit=None):
        self.policy = POLICIES[policy]
        self.theta = theta
        self.dynamic = dynamic
        self.emit = emit
        self.state_of = ["idle"] * n_exec
        self.client_of = [None] * n_exec
        self.budget_of = [None] * n_exec
        self.records = {}
        self.st = SchedState(executors=range(n_exec))
        self.pending = []
        self.n_target = 0
        self.seen = set()

    def begin_round(self, parts):
        self.pending = list(parts)
        self.n_target = len(parts)
        self.st.planned = 0
        self.seen = set()

    def _issue(self, kind, ex, now):
        self.records.setdefault(ex, []).append((kind, now, self.client_of[ex], self.budget_of[ex]))
        if self.emit is not None:
            self.emit({"t": now, "kind": "Instruction", "client": self.client_of[ex],
                       "executor": ex, "instruction": kind})
        return (kind, now, self.client_of[ex], ex, self.budget_of[ex])

    def _plan(self, now, only=None):
        if not self.pending:
            return []
        if only is None:
            got = self.policy(self.st, self.pending, self.n_target, self.theta)
        else:
            if only not in self.st.free:
                return []
            keep = self.st.free
            self.st.free = deque([only])
            got = self.policy(self.st, self.pending, self.n_target, self.theta)
            rest = self.st.free
            keep.remove(only)
            keep.extend(rest)
            self.st.free = keep
        chosen = {g[0] for g in got}
        self.pending = [p for p in self.pending if p[0] not in chosen]
        out = []
        for cid, b, ex in got:
            assert self.state_of[ex] == "idle" and cid not in self.seen
            self.seen.add(cid)
            self.state_of[ex] = "launching"
            self.client_of[ex] = cid
            self.budget_of[ex] = b
            out.append(((cid, b, ex), self._issue("launch", ex, now)))
        return out

    def kickoff(self, now):
        if self.dynamic:
            return self._plan(now)
        out = []
        for ex in [i for i, s in enumerate(self.state_of) if s == "idle"]:
            out.extend(self._plan(now, only=ex))
        return out

    def _slot(self, cid):
        for ex, c in enumerate(self.client_of):
            if c == cid and self.state_of[ex] != "idle":
                return ex
        return None

    def request(self, cid, kind, now):
        ex = self._slot(cid)
        if ex is None:
            return []
        if kind == "register":
            if self.state_of[ex] != "launching":
                return []
            self.state_of[ex] = "running"
            return [self._issue("start_training", ex, now)]
        if kind == "training_complete":
            return [self._issue("upload_model", ex, now)]
        if kind == "model_uploaded":
            self.state_of[ex] = "terminating"
            return [self._issue("terminate", ex, now)]
        raise AssertionError(kind)

    def slot_freed(self, ex, now):
        self.st.running.remove(self.budget_of[ex])
        self.state_of[ex] = "idle"
        self.client_of[ex] = None
        self.budget_of[ex] = None
        self.st.free.append(ex)
        return self._plan(now) if self.dynamic else self._plan(now, only=ex)

    def occupied(self):
        return sum(self.budget_of[i] for i, s in enumerate(self.state_of)
                   if s in ("launching", "running"))


# -- fleet config (profiles.py:76-112) --------------------------------------


@dataclass
class Config:
    theta: float = 100.0
    max_executors: int = 8
    scheduler_kind: str = "resource-aware"
    participants_per_round: int = 1
    rounds: int = 1
    aggregation: str = "sync"
    async_buffer: int = 4
    alpha: float = 2e-6
    beta: float = 1e-3
    seed: int = 1
    dynamic_parallelism: bool = True
    launch_latency: float = 0.0
    terminate_latency: float = 0.0
    upload_latency: float = 0.0

    def check(self, fleet_size=None):
        if not 0 < self.theta <= 300:
            raise ConfigError(f"theta must be in (0,300], got {self.theta}")
        if self.max_executors < 1:
            raise ConfigError("max_executors must be >= 1")
        if self.scheduler_kind not in POLICIES:
            raise ConfigError(f"unknown scheduler: {self.scheduler_kind}")
        if self.aggregation not in ("sync", "async"):
            raise ConfigError(f"unknown aggregation: {self.aggregation}")
        if self.aggregation == "async" and self.async_buffer < 1:
            raise ConfigError("async_buffer must be >= 1")
        if self.alpha <= 0 or self.beta < 0:
            raise ConfigError("cost coefficients require alpha > 0, beta >= 0")
        if fleet_size is not None and self.participants_per_round > fleet_size:
            raise ConfigError(
                f"participants_per_round {self.participants_per_round} exceeds fleet size {fleet_size}")


# -- DES (engine.py:53-230) -------------------------------------------------


def simulate_round(by_id: dict, order: list, cfg: Config, t0=0.0, trace=None, round_index=0):
    """engine.py:53-230. Returns (report dict, segment)."""
    unknown = [c for c in order if c not in by_id]
    if unknown:
        raise ConfigError(f"participants not in fleet: {unknown}")
    big = [c for c in order if by_id[c].resource_budget > cfg.theta]
    if big:
        raise ConfigError(f"clients {big} have budgets above theta={cfg.theta} and can never launch")
    work = {c: work_of(by_id[c].workload, cfg.alpha, cfg.beta) for c in order}
    ev = [] if trace is None else trace
    first = len(ev)
    mgr = Manager(cfg.max_executors, cfg.scheduler_kind, cfg.theta, cfg.dynamic_parallelism, ev.append)
    mgr.begin_round([(c, float(by_id[c].resource_budget)) for c in order])

    live = {}  # cid -> [phase_work list, phase idx, assigned]
    heap = []
    slot_of = {}
    now = t0

    def timer(t, kind, cid, ex):
        heapq.heappush(heap, (t, TIMER_RANK[kind], cid, kind, ex))

    def launched(items, t):
        for (cid, b, ex), _ in items:
            slot_of[cid] = ex
            ev.append({"t": t, "kind": "ClientLaunched", "client": cid, "executor": ex, "budget": b})
            timer(t + cfg.launch_latency, "start", cid, ex)

    def trained(cid, t):
        ex = slot_of[cid]
        ev.append({"t": t, "kind": "ClientTrainingComplete", "client": cid, "executor": ex,
                   "budget": float(by_id[cid].resource_budget)})
        mgr.request(cid, "training_complete", t)
        timer(t + cfg.upload_latency, "upload_done", cid, ex)

    def fire(kind, cid, ex, t):
        if kind == "start":
            mgr.request(cid, "register", t)
            if work[cid] <= 1e-9:
                trained(cid, t)
                return
            live[cid] = [[f * work[cid] for f, _ in by_id[cid].phases], 0, 0.0]
        elif kind == "upload_done":
            ev.append({"t": t, "kind": "ModelUploaded", "client": cid, "executor": ex,
                       "budget": float(by_id[cid].resource_budget)})
            mgr.request(cid, "model_uploaded", t)
            timer(t + cfg.terminate_latency, "slot_freed", cid, ex)
        else:
            ev.append({"t": t, "kind": "SlotFreed", "client": cid, "executor": ex})
            launched(mgr.slot_freed(ex, t), t)

    def settle(t):
        while True:
            due = []
            while heap and heap[0][0] <= t + 1e-12:
                _, rk, cid, kind, ex = heapq.heappop(heap)
                due.append((rk, cid, kind, ex))
            for cid, rc in list(live.items()):
                if rc[0][rc[1]] <= 1e-9:
                    last = rc[1] + 1 >= len(rc[0])
                    due.append((RANK["ClientTrainingComplete"] if last else RANK["PhaseCompleted"],
                                cid, "work_done", slot_of[cid]))
            if not due:
                return
            due.sort(key=lambda d: (d[0], d[1]))
            for _, cid, kind, ex in due:
                if kind != "work_done":
                    fire(kind, cid, ex, t)
                    continue
                rc = live[cid]
                if rc[1] + 1 < len(rc[0]):
                    rc[1] += 1
                    ev.append({"t": t, "kind": "PhaseCompleted", "client": cid, "executor": ex,
                               "phase": rc[1]})
                else:
                    del live[cid]
                    trained(cid, t)

    launched(mgr.kickoff(now), now)
    prev = None
    while True:
        settle(now)
        if not live and not heap:
            break
        ids = sorted(live)
        shares = water_fill([float(by_id[c].resource_budget) for c in ids],
                            [by_id[c].phases[live[c][1]][1] for c in ids])
        cur = dict(zip(ids, shares))
        for c, s in cur.items():
            live[c][2] = s
        if cur != prev:
            ev.append({"t": now, "kind": "Alloc", "alloc": cur})
            prev = dict(cur)
        assert mgr.occupied() <= cfg.theta + 1e-6
        step = min((rc[0][rc[1]] / (rc[2] / CAPACITY) for rc in live.values()), default=math.inf)
        step = min(step, heap[0][0] - now if heap else math.inf)
        if step == math.inf:
            raise RuntimeError("simulation stalled with work outstanding")
        if step > 0:
            for rc in live.values():
                rc[0][rc[1]] -= rc[2] / CAPACITY * step
                if rc[0][rc[1]] < 1e-9:
                    rc[0][rc[1]] = 0.0
            now += step
    if mgr.pending:
        raise RuntimeError(f"round ended with unlaunched participants: {mgr.pending}")
    if prev:
        ev.append({"t": now, "kind": "Alloc", "alloc": {}})
    ev.append({"t": now, "kind": "RoundComplete", "round": round_index})
    seg = ev[first:]
    return round_report(seg, round_index), seg


# -- metrics (metrics.py:31-167) ------------------------------------------


def round_report(seg, round_index=0) -> dict:
    if not seg:
        raise ValueError("empty trace")
    if not any(e["kind"] == "RoundComplete" for e in seg):
        raise ValueError("trace has no RoundComplete event")
    ups = [e["t"] for e in seg if e["kind"] == "ModelUploaded"]
    start = seg[0]["t"]
    end = max(ups) if ups else next(e["t"] for e in seg if e["kind"] == "RoundComplete")
    span = end - start

    def steps(delta):
        pts = [(start, 0.0 if delta is float else 0)]
        tot = 0.0 if delta is float else 0
        for e in seg:
            if e["kind"] == "ClientLaunched":
                tot += e["budget"] if delta is float else 1
            elif e["kind"] == "ModelUploaded":
                tot -= e["budget"] if delta is float else 1
            else:
                continue
            pts.append((e["t"], tot))
        pts.append((end, tot))
        return pts

    budget_line = steps(float)
    vac = 0.0
    for (a, v), (b, _) in zip(budget_line, budget_line[1:]):
        vac += max(0.0, CAPACITY - v) * (b - a)
    if span <= 0:
        util = 0.0
    else:
        area, pt, ptot = 0.0, start, 0.0
        for e in seg:
            if e["kind"] == "Alloc":
                area += ptot * (e["t"] - pt)
                pt, ptot = e["t"], sum(e["alloc"].values())
        area += ptot * (end - pt)
        util = area / (CAPACITY * span)
    starts, ends, budgets = {}, {}, {}
    for e in seg:
        if e["kind"] == "ClientLaunched":
            starts[e["client"]] = e["t"]
            budgets[e["client"]] = e["budget"]
        elif e["kind"] == "ModelUploaded":
            ends[e["client"]] = e["t"]
    thr = 0.0 if (len(ups) == 0 or end <= start) else len(ups) / (end - start)
    return {
        "round": round_index,
        "makespan": span,
        "utilization": util,
        "vacancy_area": vac,
        "throughput": thr,
        "parallelism_timeline": steps(int),
        "per_client_times": {c: ends[c] - starts[c] for c in ends},
        "per_client_start": starts,
        "per_client_end": ends,
        "per_client_budget": budgets,
        "degenerate": span <= 0,
    }


# -- experiment loop (engine.py:279-368) --------------------------------------


def experiment(cfg: Config, clients: list[Client], features=2, classes=4, alpha=0.5,
               train=False, lr=0.1, trace=None, keep_deltas=False) -> dict:
    cfg.check(fleet_size=len(clients))
    if cfg.rounds < 1:
        raise ConfigError("rounds must be >= 1")
    by_id = {c.client_id: c for c in clients}
    if len(by_id) != len(clients):
        raise ConfigError("duplicate client ids in fleet")
    ids = sorted(by_id)
    pick = random.Random(f"{cfg.seed}:selection")
    theta = shards = test = None
    if train:
        total = sum(c.workload.num_samples for c in clients)
        tr, test = flmath.synthetic(features, classes, max(math.ceil(total / 0.8), 10),
                                    flmath.seed_of("data", cfg.seed))
        shards = flmath.dirichlet_partition(
            tr, [(c.client_id, c.workload.num_samples) for c in clients], alpha,
            flmath.seed_of("partition", cfg.seed))
        theta = flmath.zeros_params(features, classes)
    out = {"rounds": [], "participants": [], "accuracy_series": [], "total_time": 0.0,
           "final_params": None, "deltas": []}
    now = 0.0
    for r in range(cfg.rounds):
        who = pick.sample(ids, cfg.participants_per_round)
        rep, _ = simulate_round(by_id, who, cfg, t0=now, trace=trace, round_index=r)
        out["rounds"].append(rep)
        out["participants"].append(list(who))
        end = now + rep["makespan"]
        if train:
            ds, ws, ts = [], [], []
            for cid in who:
                wl = by_id[cid].workload
                ds.append(flmath.local_sgd(theta, shards[cid], wl.num_samples, wl.batch_size, lr,
                                           classes, seed=flmath.seed_of("train", cfg.seed, r, cid)))
                ws.append(float(wl.num_samples))
                ts.append(rep["per_client_end"][cid])
            if keep_deltas:
                out["deltas"].append(ds)
            if cfg.aggregation == "sync":
                theta = flmath.weighted_average(ds, ws, theta)
                out["accuracy_series"].append((end, flmath.accuracy(theta, test)))
            else:
                seq = sorted(range(len(who)), key=lambda i: (ts[i], who[i]))
                for k in range(0, len(seq), cfg.async_buffer):
                    part = seq[k:k + cfg.async_buffer]
                    theta = flmath.weighted_average([ds[i] for i in part], [ws[i] for i in part], theta)
                    out["accuracy_series"].append((ts[part[-1]], flmath.accuracy(theta, test)))
        now = end
    out["total_time"] = now
    out["final_params"] = theta
    return out
