"""Control-plane API: cost model, client schedulers, executor manager.

Public names and semantics of fedsim's cost_model.py, scheduler.py and
executor_manager.py.  The per-round hot loop does NOT run through these
Python objects: `roundsim.run_round` drives the native C++ DES
(csrc/des.cpp), which re-implements the same policies with an incremental
sorted pending list.  These classes exist for API compatibility (callers
that step a scheduler or manager by hand) and are checked against the
oracle and the native DES in the tests.
"""

from __future__ import annotations

import ctypes as C
import enum
import logging
from collections import deque
from dataclasses import dataclass, field

from . import _abi
from .errors import ConfigError
from .spec import WorkloadSpec

log = logging.getLogger(__name__)

CAPACITY = 100.0
_EPS = 1e-9


# ---- cost model (cost_model.py:18-102) ------------------------------------


@dataclass(frozen=True)
class CostCoefficients:
    alpha: float = 2e-6
    beta: float = 1e-3

    def __post_init__(self):
        if self.alpha <= 0:
            raise ConfigError(f"alpha must be > 0, got {self.alpha}")
        if self.beta < 0:
            raise ConfigError(f"beta must be >= 0, got {self.beta}")


def work_units(w: WorkloadSpec, c: CostCoefficients) -> float:
    """Seconds-at-full-capacity of one local pass (native, same fp64 order)."""
    return _abi.lib.fedhc_work_units(w.num_samples, w.batch_size, w.model_layers, w.seq_len,
                                     float(w.extra_model_factor), float(c.alpha), float(c.beta))


def maxmin_allocate(caps: list[float], demands: list[float], capacity: float = CAPACITY) -> list[float]:
    """Capped max-min (water-filling) shares; native implementation."""
    if len(caps) != len(demands):
        raise ConfigError("caps and demands must have equal length")
    n = len(caps)
    if n == 0:
        return []
    for cap, dem in zip(caps, demands):
        if not 0 < cap <= 100:
            raise ConfigError(f"cap {cap} outside (0,100]")
        if not 0 < dem <= 100:
            raise ConfigError(f"demand {dem} outside (0,100]")
    arr = C.c_double * n
    out = arr()
    _abi.check(_abi.lib.fedhc_maxmin_allocate(arr(*map(float, caps)), arr(*map(float, demands)), n,
                                              float(capacity), out))
    return list(out)


def rate(assigned: float, demand: float = CAPACITY) -> float:
    if not 0 < assigned <= demand <= 100:
        raise ConfigError(f"need 0 < assigned <= demand <= 100, got {assigned}, {demand}")
    return assigned / CAPACITY


def solo_time(budget: float, demand_profile, total_work: float) -> float:
    return sum(p.work_fraction * total_work / rate(min(budget, p.demand)) for p in demand_profile)


# ---- schedulers (scheduler.py:17-130) --------------------------------------


@dataclass(frozen=True)
class Participant:
    client_id: str
    resource_budget: float


@dataclass(frozen=True)
class ScheduleEntry:
    client_id: str
    resource_budget: float
    executor_id: int


@dataclass
class SchedulerState:
    running_budgets: list[float] = field(default_factory=list)
    planned_count: int = 0
    available_executors: deque[int] = field(default_factory=deque)

    def running_total(self) -> float:
        return sum(self.running_budgets)

    def admit(self, cand: Participant, theta: float) -> ScheduleEntry | None:
        """Accept iff the budget fits under theta and an executor is idle."""
        if not self.available_executors or cand.resource_budget + self.running_total() > theta + _EPS:
            return None
        slot = self.available_executors.popleft()
        self.running_budgets.append(cand.resource_budget)
        self.planned_count += 1
        return ScheduleEntry(cand.client_id, cand.resource_budget, slot)

    def has_room(self, n_participants: int, theta: float) -> bool:
        return self.planned_count < n_participants and self.running_total() < theta - _EPS


def schedule_resource_aware(state: SchedulerState, pending: list[Participant], n_participants: int,
                            theta: float) -> list[ScheduleEntry]:
    """Double-pointer policy (PAPER Alg. 1): smallest and largest budgets alternately.

    A left rejection ends the pass; a right rejection only retires the right
    pointer.
    """
    ranked = sorted(pending, key=lambda p: (p.resource_budget, p.client_id))
    lo, hi, use_hi = 0, len(ranked) - 1, True
    taken: list[ScheduleEntry] = []
    while state.has_room(n_participants, theta) and lo <= hi:
        got = state.admit(ranked[lo], theta)
        if got is None:
            break
        taken.append(got)
        lo += 1
        if not state.has_room(n_participants, theta) or lo > hi or not use_hi:
            continue
        got = state.admit(ranked[hi], theta)
        if got is None:
            use_hi = False
        else:
            taken.append(got)
            hi -= 1
    return taken


def schedule_greedy(state: SchedulerState, pending: list[Participant], n_participants: int,
                    theta: float) -> list[ScheduleEntry]:
    """FIFO with strict head-of-line blocking."""
    taken: list[ScheduleEntry] = []
    for cand in pending:
        if not state.has_room(n_participants, theta):
            break
        got = state.admit(cand, theta)
        if got is None:
            break
        taken.append(got)
    return taken


SCHEDULERS = {"resource-aware": schedule_resource_aware, "greedy": schedule_greedy}


# ---- executor manager (executor_manager.py:28-238) -------------------------


class Lifecycle(enum.Enum):
    IDLE = "idle"
    LAUNCHING = "launching"
    RUNNING = "running"
    TERMINATING = "terminating"


class InstructionKind(enum.Enum):
    LAUNCH = "launch"
    START_TRAINING = "start_training"
    UPLOAD_MODEL = "upload_model"
    TERMINATE = "terminate"


class RequestKind(enum.Enum):
    REGISTER = "register"
    TRAINING_COMPLETE = "training_complete"
    MODEL_UPLOADED = "model_uploaded"


@dataclass(frozen=True)
class Instruction:
    kind: InstructionKind
    issued_at: float
    client_id: str
    executor_id: int
    budget: float | None = None


@dataclass(frozen=True)
class ClientRequest:
    client_id: str
    kind: RequestKind


@dataclass
class ExecutorSlot:
    executor_id: int
    lifecycle: Lifecycle = Lifecycle.IDLE
    client_id: str | None = None
    budget: float | None = None


@dataclass
class RecordTable:
    capacity: int
    rows: dict[int, deque[Instruction]] = field(default_factory=dict)

    def append(self, instr: Instruction) -> None:
        self.rows.setdefault(instr.executor_id, deque()).append(instr)


# request kind -> (required lifecycle or None, next lifecycle or None, instruction)
_TRANSITIONS = {
    RequestKind.REGISTER: (Lifecycle.LAUNCHING, Lifecycle.RUNNING, InstructionKind.START_TRAINING),
    RequestKind.TRAINING_COMPLETE: (None, None, InstructionKind.UPLOAD_MODEL),
    RequestKind.MODEL_UPLOADED: (None, Lifecycle.TERMINATING, InstructionKind.TERMINATE),
}


class ExecutorManager:
    """Executor-slot lifecycles, per-slot instruction FIFO and status monitor.

    Single logical owner; in this framework an executor slot is a
    green-context SM partition and a slot's budget is
    immutable for one occupancy.
    """

    def __init__(self, max_executors: int, scheduler_kind: str, theta: float, dynamic_parallelism: bool = True,
                 trace=None):
        self.max_executors = max_executors
        self.scheduler_fn = SCHEDULERS[scheduler_kind]
        self.theta = theta
        self.dynamic_parallelism = dynamic_parallelism
        self.trace = trace
        self.slots = {i: ExecutorSlot(i) for i in range(max_executors)}
        self.record_table = RecordTable(capacity=max_executors)
        self.state = SchedulerState(available_executors=deque(range(max_executors)))
        self.pending: list[Participant] = []
        self.n_participants = 0
        self._launched: set[str] = set()

    def begin_round(self, participants: list[Participant]) -> None:
        self.pending = list(participants)
        self.n_participants = len(participants)
        self.state.planned_count = 0
        self._launched = set()

    def kickoff(self, now: float):
        if self.dynamic_parallelism:
            return self._schedule(now)
        out = []
        for slot in [s.executor_id for s in self.slots.values() if s.lifecycle is Lifecycle.IDLE]:
            out += self._schedule(now, only_executor=slot)
        return out

    def on_request(self, req: ClientRequest, now: float) -> list[Instruction]:
        slot = self._slot_of(req.client_id)
        if slot is None:
            log.warning("request %s from %s with no slot; dropped", req.kind, req.client_id)
            return []
        need, nxt, kind = _TRANSITIONS[req.kind]
        if need is not None and slot.lifecycle is not need:
            log.warning("register from %s in %s; dropped", req.client_id, slot.lifecycle)
            return []
        if nxt is not None:
            slot.lifecycle = nxt
        return [self._issue(kind, slot, now)]

    def on_slot_freed(self, executor_id: int, now: float):
        slot = self.slots[executor_id]
        self.state.running_budgets.remove(slot.budget)
        slot.lifecycle, slot.client_id, slot.budget = Lifecycle.IDLE, None, None
        self.state.available_executors.append(executor_id)
        return self._schedule(now, None if self.dynamic_parallelism else executor_id)

    def occupied_budget(self) -> float:
        return sum(s.budget for s in self.slots.values() if s.lifecycle in (Lifecycle.LAUNCHING, Lifecycle.RUNNING))

    def all_idle(self) -> bool:
        return all(s.lifecycle is Lifecycle.IDLE for s in self.slots.values())

    def _slot_of(self, client_id: str) -> ExecutorSlot | None:
        return next((s for s in self.slots.values()
                     if s.client_id == client_id and s.lifecycle is not Lifecycle.IDLE), None)

    def _issue(self, kind: InstructionKind, slot: ExecutorSlot, now: float) -> Instruction:
        instr = Instruction(kind, now, slot.client_id, slot.executor_id, slot.budget)
        self.record_table.append(instr)
        if self.trace is not None:
            self.trace({"t": now, "kind": "Instruction", "client": instr.client_id, "executor": instr.executor_id,
                        "instruction": kind.value})
        return instr

    def _schedule(self, now: float, only_executor: int | None = None):
        if not self.pending:
            return []
        st = self.state
        if only_executor is None:
            entries = self.scheduler_fn(st, self.pending, self.n_participants, self.theta)
        else:
            # fixed parallelism: offer only the freed executor
            if only_executor not in st.available_executors:
                return []
            others = st.available_executors
            others.remove(only_executor)
            st.available_executors = deque([only_executor])
            entries = self.scheduler_fn(st, self.pending, self.n_participants, self.theta)
            others.extend(st.available_executors)
            st.available_executors = others
        chosen = {e.client_id for e in entries}
        self.pending = [p for p in self.pending if p.client_id not in chosen]
        launches = []
        for entry in entries:
            slot = self.slots[entry.executor_id]
            assert slot.lifecycle is Lifecycle.IDLE
            assert entry.client_id not in self._launched, "client relaunched in round"
            self._launched.add(entry.client_id)
            slot.lifecycle, slot.client_id, slot.budget = Lifecycle.LAUNCHING, entry.client_id, entry.resource_budget
            launches.append((entry, self._issue(InstructionKind.LAUNCH, slot, now)))
        return launches
