"""Round simulation and per-client runtime accounting.

`run_round` has the signature and outputs of fedsim's engine.run_round
(engine.py:53-230) but executes in the native C++ DES (csrc/des.cpp):
selection order in, RoundReport + event trace out, bit-identical to the
reference.  The trace-analysis functions (metrics.py:31-178 API) are pure
Python functions of a trace so that saved JSONL traces can be re-analysed.
"""

from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from .errors import ConfigError, TraceError
from .spec import ClientProfile, FleetConfig

CAPACITY = 100.0

KIND_RANK = {
    "ClientLaunched": 0,
    "PhaseCompleted": 1,
    "ClientTrainingComplete": 2,
    "ModelUploaded": 3,
    "SlotFreed": 4,
    "RoundComplete": 5,
}
_INSTR = ("launch", "start_training", "upload_model", "terminate")
_EVENT = np.dtype([("t", "<f8"), ("kind", "<i4"), ("client", "<i4"), ("executor", "<i4"), ("aux", "<i4"),
                   ("budget", "<f8"), ("alloc_off", "<i8"), ("alloc_len", "<i4"), ("pad_", "<i4")])
assert _EVENT.itemsize == C.sizeof(_abi.DesEvent)


@dataclass
class RoundReport:
    round_index: int
    makespan: float
    utilization: float
    vacancy_area: float
    throughput: float
    parallelism_timeline: list[tuple[float, int]]
    per_client_times: dict[str, float]
    per_client_start: dict[str, float] = field(default_factory=dict)
    per_client_end: dict[str, float] = field(default_factory=dict)
    per_client_budget: dict[str, float] = field(default_factory=dict)
    degenerate: bool = False

    def to_dict(self) -> dict:
        return {
            "round": self.round_index,
            "makespan_s": self.makespan,
            "utilization": self.utilization,
            "vacancy_area": self.vacancy_area,
            "throughput": self.throughput,
            "n_clients": len(self.per_client_times),
        }


class RoundSimulator:
    """Reusable native DES handle plus the ctypes views of one fleet.

    Build it once per fleet (it marshals the profiles once); `run` then costs
    one native call per round.
    """

    def __init__(self, fleet: dict[str, ClientProfile]):
        self.ids = list(fleet)
        self.index = {cid: i for i, cid in enumerate(self.ids)}
        n = len(self.ids)
        self._clients = (_abi.DesClient * max(n, 1))()
        self._phase_store = []
        for i, cid in enumerate(self.ids):
            p = fleet[cid]
            w = p.workload
            fr = (C.c_double * len(p.demand_profile))(*[ph.work_fraction for ph in p.demand_profile])
            dm = (C.c_double * len(p.demand_profile))(*[ph.demand for ph in p.demand_profile])
            self._phase_store += [fr, dm]
            self._clients[i] = _abi.DesClient(p.resource_budget, w.num_samples, w.batch_size, w.model_layers,
                                              w.seq_len, float(w.extra_model_factor), len(p.demand_profile), fr, dm)
        self._id_bytes = [cid.encode() for cid in self.ids]
        self._id_arr = (C.c_char_p * max(n, 1))(*self._id_bytes)
        self.budget = {cid: fleet[cid].resource_budget for cid in self.ids}
        self._sim = _abi.lib.fedhc_des_create()
        self._lean_cap, self._lean_key, self._lean_conf = 0, None, None

    def __del__(self):
        sim = getattr(self, "_sim", None)
        if sim:
            _abi.lib.fedhc_des_destroy(sim)
            self._sim = None

    def run(self, participant_ids: list[str], cfg: FleetConfig, t0: float = 0.0, round_index: int = 0,
            want_trace: bool = True):
        missing = [cid for cid in participant_ids if cid not in self.index]
        if missing:
            raise ConfigError(f"participants not in fleet: {missing}")
        too_big = [cid for cid in participant_ids if self.budget[cid] > cfg.theta]
        if too_big:
            raise ConfigError(f"clients {too_big} have budgets above theta={cfg.theta} and can never launch")
        n = len(participant_ids)
        index = self.index
        order = (C.c_int32 * max(n, 1))(*[index[c] for c in participant_ids])
        conf = _abi.DesConfig(float(cfg.theta), int(cfg.max_executors),
                              0 if cfg.scheduler_kind == "resource-aware" else 1, int(bool(cfg.dynamic_parallelism)),
                              float(cfg.alpha), float(cfg.beta), float(cfg.launch_latency),
                              float(cfg.terminate_latency), float(cfg.upload_latency))
        if cfg.scheduler_kind not in ("resource-aware", "greedy"):
            raise KeyError(cfg.scheduler_kind)
        starts = (C.c_double * max(n, 1))()
        ends = (C.c_double * max(n, 1))()
        rep = _abi.DesReport()
        _abi.check(_abi.lib.fedhc_des_run_round(self._sim, self._clients, self._id_arr, order, n, C.byref(conf),
                                                float(t0), int(round_index), 1, starts, ends, C.byref(rep)))
        ev = C.POINTER(_abi.DesEvent)()
        ac = C.POINTER(C.c_int32)()
        ash = C.POINTER(C.c_double)()
        pt = C.POINTER(C.c_double)()
        pn = C.POINTER(C.c_int32)()
        npar = C.c_int()
        _abi.check(_abi.lib.fedhc_des_trace(self._sim, C.byref(ev), C.byref(ac), C.byref(ash), C.byref(pt),
                                            C.byref(pn), C.byref(npar)))
        pid = participant_ids
        events = np.ctypeslib.as_array(C.cast(ev, C.POINTER(C.c_uint8)), shape=(rep.n_events * _EVENT.itemsize,))
        events = events.view(_EVENT)
        kinds, who = events["kind"], events["client"]
        launch_order = who[kinds == _abi.EV_LAUNCHED].tolist()
        upload_order = who[kinds == _abi.EV_UPLOADED].tolist()
        st = np.ctypeslib.as_array(starts, shape=(max(n, 1),))
        en = np.ctypeslib.as_array(ends, shape=(max(n, 1),))
        st_l, en_l = st.tolist(), en.tolist()
        par = list(zip(np.ctypeslib.as_array(pt, shape=(npar.value,)).tolist(),
                       np.ctypeslib.as_array(pn, shape=(npar.value,)).tolist())) if npar.value else []
        seg = [self._event_dict(ev[k], pid, ac, ash) for k in range(rep.n_events)] if want_trace else None
        report = RoundReport(
            round_index=round_index,
            makespan=rep.makespan,
            utilization=rep.utilization,
            vacancy_area=rep.vacancy_area,
            throughput=rep.throughput,
            parallelism_timeline=par,
            per_client_times={pid[i]: en_l[i] - st_l[i] for i in upload_order},
            per_client_start={pid[i]: st_l[i] for i in launch_order},
            per_client_end={pid[i]: en_l[i] for i in upload_order},
            per_client_budget={pid[i]: float(self.budget[pid[i]]) for i in launch_order},
            degenerate=bool(rep.degenerate),
        )
        return report, seg

    def run_lean(self, order: np.ndarray, participant_ids: list[str], cfg: FleetConfig, t0: float = 0.0,
                 round_index: int = 0) -> "LeanRoundReport":
        """`run` for the serving loop: `order` are this simulator's client indices (int32) of participants the
        caller has already validated; buffers and the config block are reused, and the per-client dicts of
        the RoundReport are built only if someone asks (LeanRoundReport.full / attribute access)."""
        n = int(order.shape[0])
        if n > self._lean_cap:
            self._lean_cap = max(n, 2 * self._lean_cap)
            self._lean_order = (C.c_int32 * self._lean_cap)()
            self._lean_starts = (C.c_double * self._lean_cap)()
            self._lean_ends = (C.c_double * self._lean_cap)()
        C.memmove(self._lean_order, np.ascontiguousarray(order, dtype=np.int32).ctypes.data, 4 * n)
        key = (cfg.theta, cfg.max_executors, cfg.scheduler_kind, cfg.dynamic_parallelism, cfg.alpha, cfg.beta,
               cfg.launch_latency, cfg.terminate_latency, cfg.upload_latency)
        if self._lean_key != key:
            if cfg.scheduler_kind not in ("resource-aware", "greedy"):
                raise KeyError(cfg.scheduler_kind)
            self._lean_conf = _abi.DesConfig(float(cfg.theta), int(cfg.max_executors),
                                             0 if cfg.scheduler_kind == "resource-aware" else 1,
                                             int(bool(cfg.dynamic_parallelism)), float(cfg.alpha), float(cfg.beta),
                                             float(cfg.launch_latency), float(cfg.terminate_latency),
                                             float(cfg.upload_latency))
            self._lean_key = key
        rep = _abi.DesReport()
        _abi.check(_abi.lib.fedhc_des_run_round(self._sim, self._clients, self._id_arr, self._lean_order, n,
                                                C.byref(self._lean_conf), float(t0), int(round_index), 1,
                                                self._lean_starts, self._lean_ends, C.byref(rep)))
        ev = C.POINTER(_abi.DesEvent)()
        ac = C.POINTER(C.c_int32)()
        ash = C.POINTER(C.c_double)()
        pt = C.POINTER(C.c_double)()
        pn = C.POINTER(C.c_int32)()
        npar = C.c_int()
        _abi.check(_abi.lib.fedhc_des_trace(self._sim, C.byref(ev), C.byref(ac), C.byref(ash), C.byref(pt),
                                            C.byref(pn), C.byref(npar)))
        events = np.ctypeslib.as_array(C.cast(ev, C.POINTER(C.c_uint8)), shape=(rep.n_events * _EVENT.itemsize,))
        events = events.view(_EVENT)
        kinds, who = events["kind"], events["client"]
        return LeanRoundReport(
            round_index, rep.makespan, rep.utilization, rep.vacancy_area, rep.throughput, bool(rep.degenerate),
            participant_ids, who[kinds == _abi.EV_LAUNCHED].copy(), who[kinds == _abi.EV_UPLOADED].copy(),
            np.ctypeslib.as_array(self._lean_starts, shape=(self._lean_cap,))[:n].copy(),
            np.ctypeslib.as_array(self._lean_ends, shape=(self._lean_cap,))[:n].copy(),
            np.ctypeslib.as_array(pt, shape=(npar.value,)).copy() if npar.value else None,
            np.ctypeslib.as_array(pn, shape=(npar.value,)).copy() if npar.value else None,
            self.budget)

    @staticmethod
    def _event_dict(e, pid, ac, ash) -> dict:
        kind = e.kind
        if kind == _abi.EV_INSTRUCTION:
            return {"t": e.t, "kind": "Instruction", "client": pid[e.client], "executor": e.executor,
                    "instruction": _INSTR[e.aux]}
        if kind == _abi.EV_ALLOC:
            off = e.alloc_off
            return {"t": e.t, "kind": "Alloc", "alloc": {pid[ac[off + j]]: ash[off + j] for j in range(e.alloc_len)}}
        if kind == _abi.EV_ROUND_COMPLETE:
            return {"t": e.t, "kind": "RoundComplete", "round": e.aux}
        if kind == _abi.EV_PHASE:
            return {"t": e.t, "kind": "PhaseCompleted", "client": pid[e.client], "executor": e.executor,
                    "phase": e.aux}
        if kind == _abi.EV_SLOT_FREED:
            return {"t": e.t, "kind": "SlotFreed", "client": pid[e.client], "executor": e.executor}
        name = {_abi.EV_LAUNCHED: "ClientLaunched", _abi.EV_TRAINED: "ClientTrainingComplete",
                _abi.EV_UPLOADED: "ModelUploaded"}[kind]
        return {"t": e.t, "kind": name, "client": pid[e.client], "executor": e.executor, "budget": e.budget}


class LeanRoundReport:
    """A RoundReport whose per-client dicts are built on first use (the scalar fields are plain attributes)."""

    def __init__(self, round_index, makespan, utilization, vacancy_area, throughput, degenerate, pid, launch, upload,
                 starts, ends, par_t, par_n, budget):
        self.round_index, self.makespan, self.utilization = round_index, makespan, utilization
        self.vacancy_area, self.throughput, self.degenerate = vacancy_area, throughput, degenerate
        self._raw = (pid, launch, upload, starts, ends, par_t, par_n, budget)
        self._full = None

    def end_times(self) -> np.ndarray:
        """ModelUploaded times in participant order (per_client_end without the dict)."""
        return self._raw[4]

    def full(self) -> RoundReport:
        if self._full is None:
            pid, launch, upload, starts, ends, par_t, par_n, budget = self._raw
            st_l, en_l = starts.tolist(), ends.tolist()
            lo, up = launch.tolist(), upload.tolist()
            self._full = RoundReport(
                round_index=self.round_index, makespan=self.makespan, utilization=self.utilization,
                vacancy_area=self.vacancy_area, throughput=self.throughput,
                parallelism_timeline=list(zip(par_t.tolist(), par_n.tolist())) if par_t is not None else [],
                per_client_times={pid[i]: en_l[i] - st_l[i] for i in up},
                per_client_start={pid[i]: st_l[i] for i in lo},
                per_client_end={pid[i]: en_l[i] for i in up},
                per_client_budget={pid[i]: float(budget[pid[i]]) for i in lo},
                degenerate=self.degenerate)
        return self._full

    def __getattr__(self, name):
        if name.startswith("_"):
            raise AttributeError(name)
        return getattr(self.full(), name)


def run_round(fleet: dict[str, ClientProfile], participant_ids: list[str], cfg: FleetConfig, t0: float = 0.0,
              trace: list[dict] | None = None, round_index: int = 0) -> tuple[RoundReport, list[dict]]:
    """engine.run_round drop-in: one round of the native DES; appends to `trace` if given."""
    report, seg = RoundSimulator(fleet).run(participant_ids, cfg, t0, round_index, want_trace=True)
    if trace is not None:
        trace.extend(seg)
    return report, seg


# ---- trace analysis (metrics.py API) -----------------------------------------


def _round_bounds(trace: list[dict]) -> tuple[float, float]:
    if not trace:
        raise TraceError("empty trace")
    done = [e["t"] for e in trace if e["kind"] == "RoundComplete"]
    if not done:
        raise TraceError("trace has no RoundComplete event")
    uploads = [e["t"] for e in trace if e["kind"] == "ModelUploaded"]
    return trace[0]["t"], (max(uploads) if uploads else done[0])


def _step_function(trace, weight, zero):
    start, end = _round_bounds(trace)
    level = zero
    points = [(start, zero)]
    for e in trace:
        sign = {"ClientLaunched": 1, "ModelUploaded": -1}.get(e["kind"])
        if sign is None:
            continue
        level = level + weight(e) if sign > 0 else level - weight(e)
        points.append((e["t"], level))
    points.append((end, level))
    return points


def budget_timeline(trace: list[dict]) -> list[tuple[float, float]]:
    return _step_function(trace, lambda e: e["budget"], 0.0)


def parallelism_timeline(trace: list[dict]) -> list[tuple[float, int]]:
    return _step_function(trace, lambda e: 1, 0)


def vacancy_area(trace: list[dict]) -> float:
    pts = budget_timeline(trace)
    area = 0.0
    for (a, v), (b, _) in zip(pts, pts[1:]):
        area += max(0.0, CAPACITY - v) * (b - a)
    return area


def utilization(trace: list[dict]) -> float:
    start, end = _round_bounds(trace)
    span = end - start
    if span <= 0:
        return 0.0
    area, prev_t, prev_total = 0.0, start, 0.0
    for e in trace:
        if e["kind"] == "Alloc":
            area += prev_total * (e["t"] - prev_t)
            prev_t, prev_total = e["t"], sum(e["alloc"].values())
    area += prev_total * (end - prev_t)
    return area / (CAPACITY * span)


def per_client_times(trace: list[dict]):
    starts, ends, budgets = {}, {}, {}
    for e in trace:
        if e["kind"] == "ClientLaunched":
            starts[e["client"]], budgets[e["client"]] = e["t"], e["budget"]
        elif e["kind"] == "ModelUploaded":
            ends[e["client"]] = e["t"]
    return {c: ends[c] - starts[c] for c in ends}, starts, ends, budgets


def throughput(trace: list[dict]) -> float:
    start, end = _round_bounds(trace)
    done = sum(1 for e in trace if e["kind"] == "ModelUploaded")
    return 0.0 if (done == 0 or end <= start) else done / (end - start)


def build_round_report(trace: list[dict], round_index: int = 0) -> RoundReport:
    start, end = _round_bounds(trace)
    walls, starts, ends, budgets = per_client_times(trace)
    return RoundReport(round_index, end - start, utilization(trace), vacancy_area(trace), throughput(trace),
                       parallelism_timeline(trace), walls, starts, ends, budgets, degenerate=(end - start) <= 0)


def write_trace_jsonl(trace: list[dict], path) -> None:
    with open(path, "w") as fh:
        fh.writelines(json.dumps(e, sort_keys=True) + "\n" for e in trace)


def read_trace_jsonl(path) -> list[dict]:
    with open(path) as fh:
        return [json.loads(line) for line in fh if line.strip()]
