"""Experiment loop with an HBM-resident federation -- drop-in for engine.run_experiment.

`run_experiment` keeps the reference's semantics (engine.py:279-368):
seeded selection (`random.Random(f"{seed}:selection").sample`), the round
DES, per-client local SGD from the round-start model, then sync FedAvg or
async buffered aggregation in (per_client_end, id) order, then accuracy.

What changes is where the work runs.  `DeviceFederation` uploads every
client's shard and the test set to HBM once; each round then costs
  host:   selection + native DES + PCG64 batch permutations (the data plan),
  device: ONE fedhc_local_train launch for all participants (one CTA per
          client), ONE fedhc_fedavg launch per aggregation and ONE
          fedhc_eval launch per accuracy point,
with only the permutations (int32) copied in and the accuracy count copied
out.  Clients of a round train concurrently because every participant starts
from the same round-start params (engine.py:336-347).
"""

from __future__ import annotations

import ctypes as C
import json
import math
import os
import random
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _abi
from .devicedata import reference_federation
from .errors import AggregationError, ConfigError
from .roundsim import LeanRoundReport, RoundReport, RoundSimulator
from .spec import ClientProfile, FleetConfig
from .training import (Dataset, DatasetShard, check_aggregation, count_correct, device, fedavg_device,
                       init_params, n_permutations, native_permutations,
                       split_supported, stable_seed, stream_ptr, train_launch, train_sms_per_client, x_split)


@dataclass
class TrainParams:
    enabled: bool = True
    lr: float = 0.1


@dataclass
class DataParams:
    features: int = 2
    classes: int = 4
    alpha: float = 0.5


@dataclass
class ExperimentReport:
    rounds: list[RoundReport] = field(default_factory=list)
    participants: list[list[str]] = field(default_factory=list)
    accuracy_series: list[tuple[float, float]] = field(default_factory=list)
    total_time: float = 0.0
    final_params: np.ndarray | None = None

    def mean_round_time(self) -> float:
        return sum(r.makespan for r in self.rounds) / len(self.rounds) if self.rounds else 0.0

    def accuracy_at(self, sim_time: float) -> float:
        acc = 0.0
        for t, a in self.accuracy_series:
            if t > sim_time:
                break
            acc = a
        return acc

    def to_json(self) -> str:
        return json.dumps({"rounds": [r.to_dict() for r in self.rounds], "participants": self.participants,
                           "accuracy_series": self.accuracy_series, "total_time": self.total_time}, sort_keys=True)


class DeviceFederation:
    """All client shards + the test set resident in HBM; batched round kernels.

    Shards are packed back to back in one fp32 [sum n_i, F] buffer (labels
    int32); a client's descriptor points at its slice.  Only the round's
    permutations travel host->device per round (pinned staging).
    """

    def __init__(self, shards: dict[str, DatasetShard], test: Dataset, n_features: int, n_classes: int):
        dev = device()
        self.n_features, self.n_classes = n_features, n_classes
        self.P = n_features * n_classes + n_classes
        ids = list(shards)
        sizes = [len(shards[c].labels) for c in ids]
        self.offset, off = {}, 0
        for cid, n in zip(ids, sizes):
            self.offset[cid] = (off, n)
            off += n
        total = max(off, 1)
        x = np.zeros((total, n_features), dtype=np.float32)
        y = np.zeros(total, dtype=np.int32)
        for cid in ids:
            o, n = self.offset[cid]
            if n:
                x[o:o + n] = shards[cid].features
                y[o:o + n] = shards[cid].labels
        self.x = torch.from_numpy(x).to(dev)
        self.y = torch.from_numpy(y).to(dev)
        self.x_test = torch.from_numpy(np.ascontiguousarray(test.features, dtype=np.float32)).to(dev)
        self.y_test = torch.from_numpy(np.ascontiguousarray(test.labels, dtype=np.int32)).to(dev)
        self.n_test = len(test.labels)
        self._cap = 0
        self._pinned = None
        self._perm_dev = None
        self.x_split = x_split(self.x) if split_supported(n_features, n_classes) else None

    @classmethod
    def from_arrays(cls, x: torch.Tensor, y: torch.Tensor, offsets: dict[str, tuple[int, int]],
                    x_test: torch.Tensor, y_test: torch.Tensor, n_classes: int) -> "DeviceFederation":
        """Wrap already-resident device tensors (e.g. on-device synthetic data)."""
        self = cls.__new__(cls)
        self.n_features, self.n_classes = int(x.shape[1]), n_classes
        self.P = self.n_features * n_classes + n_classes
        self.x, self.y, self.offset = x, y, dict(offsets)
        self.x_test, self.y_test, self.n_test = x_test, y_test, int(y_test.shape[0])
        self._cap, self._pinned, self._perm_dev = 0, None, None
        self.x_split = x_split(self.x) if split_supported(self.n_features, n_classes) else None
        return self

    def launch_train(self, desc_ptr: int, k: int, params: torch.Tensor, max_batch: int,
                     stream: int | None = None) -> None:
        """fedhc_local_train(_split) for k device descriptors pointing into this federation's rows."""
        train_launch(desc_ptr, k, params.data_ptr(), self.n_features, self.n_classes, max_batch, self.x,
                     self.x_split, stream)

    # ---- per-round plan (host) ------------------------------------------
    def plan_meta(self, participants: list[str], workloads, seeds):
        """Per participant (offset into the packed permutation buffer, n_rows, steps, batch) + native args."""
        meta, at = [], 0
        rows, perms, rseeds = [], [], []
        for cid, wl, sd in zip(participants, workloads, seeds):
            _, n = self.offset[cid]
            k = n_permutations(n, wl.num_samples, wl.batch_size)
            meta.append((at, n, math.ceil(wl.num_samples / wl.batch_size), wl.batch_size))
            rows.append(n)
            perms.append(k)
            rseeds.append(stable_seed("local_train", sd))
            at += n * k
        return meta, at, (rseeds, rows, perms)

    def plan(self, participants: list[str], workloads, seeds) -> tuple[np.ndarray, list[tuple[int, int, int, int]]]:
        """PCG64 batch permutations for every participant, packed (int32, host)."""
        meta, total, (rseeds, rows, perms) = self.plan_meta(participants, workloads, seeds)
        return native_permutations(rseeds, rows, perms), meta

    def _ensure_plan_capacity(self, n: int):
        if getattr(self, "_copied", None) is not None:
            self._copied.synchronize()  # previous H2D must finish before the pinned buffer is reused
        if n > self._cap:
            self._cap = max(n, 2 * self._cap)
            self._pinned = torch.empty(self._cap, dtype=torch.int32, pin_memory=True)
            self._perm_dev = torch.empty(self._cap, dtype=torch.int32, device=self.x.device)

    def stage_plan(self, participants: list[str], workloads, seeds):
        """Generate the permutations straight into pinned memory and start the H2D copy."""
        meta, total, (rseeds, rows, perms) = self.plan_meta(participants, workloads, seeds)
        self._ensure_plan_capacity(max(total, 1))
        if total:
            native_permutations(rseeds, rows, perms, out=self._pinned.numpy())
            self._perm_dev[:total].copy_(self._pinned[:total], non_blocking=True)
            self._copied = torch.cuda.Event()
            self._copied.record()
        return meta, total * 4

    def upload_plan(self, packed: np.ndarray) -> torch.Tensor:
        n = packed.shape[0]
        self._ensure_plan_capacity(max(n, 1))
        if n:
            self._pinned[:n].numpy()[:] = packed
            self._perm_dev[:n].copy_(self._pinned[:n], non_blocking=True)
            self._copied = torch.cuda.Event()
            self._copied.record()
        return self._perm_dev

    def descriptor_array(self, participants, meta, lr: float, deltas: torch.Tensor,
                         perm_base: int | None = None) -> np.ndarray:
        """fedhc_client records for the round as a numpy structured array (vectorised packing)."""
        k = len(participants)
        rec = np.zeros(k, dtype=CLIENT_DTYPE)
        if k == 0:
            return rec
        F = self.n_features
        off = np.fromiter((self.offset[c][0] for c in participants), dtype=np.int64, count=k)
        m = np.asarray(meta, dtype=np.int64).reshape(k, 4)
        pb = self._perm_dev.data_ptr() if perm_base is None else perm_base
        rec["x"] = self.x.data_ptr() + off * (F * 4)
        rec["y"] = self.y.data_ptr() + off * 4
        rec["perm"] = pb + m[:, 0] * 4
        rec["n_rows"], rec["n_batches"], rec["batch_size"] = m[:, 1], m[:, 2], m[:, 3]
        rec["lr"] = lr
        rec["delta"] = deltas.data_ptr() + np.arange(k, dtype=np.int64) * (deltas.stride(0) * 4)
        return rec

    def descriptors(self, participants, meta, lr: float, deltas: torch.Tensor, rows=None) -> torch.Tensor:
        """fedhc_client records on the device; record i writes its delta into deltas[rows[i]] (default i)."""
        descs = (_abi.Client * max(len(participants), 1))()
        xb, yb, pb = self.x.data_ptr(), self.y.data_ptr(), self._perm_dev.data_ptr() if self._perm_dev is not None \
            else 0
        F = self.n_features
        for i, (cid, (at, n, steps, bs)) in enumerate(zip(participants, meta)):
            o, _ = self.offset[cid]
            descs[i] = _abi.Client(xb + o * F * 4, yb + o * 4, pb + at * 4, n, steps, bs, float(lr),
                                   deltas[i if rows is None else rows[i]].data_ptr())
        raw = torch.frombuffer(bytearray(descs), dtype=torch.uint8).pin_memory()
        return raw.to(self.x.device, non_blocking=True)

    # ---- device work --------------------------------------------------
    def train(self, params: torch.Tensor, participants: list[str], workloads, lr: float, seeds,
              deltas: torch.Tensor | None = None) -> torch.Tensor:
        """Local SGD for all participants in one launch; returns fp32 deltas [K, P]."""
        k = len(participants)
        if deltas is None:
            deltas = delta_buffer(k, self.P, self.x.device)
        meta, _ = self.stage_plan(participants, workloads, seeds)
        d_desc = self.descriptors(participants, meta, lr, deltas)
        max_batch = max((wl.batch_size for wl in workloads), default=1)
        self.launch_train(d_desc.data_ptr(), k, params, max_batch)
        self._keepalive = d_desc
        return deltas

    def aggregate(self, params: torch.Tensor, deltas: torch.Tensor, weights: list[float],
                  rows: list[int] | None = None) -> torch.Tensor:
        """params <- params + sum_i (w_i / sum w) * deltas[rows[i]] (fp64, list order), in place."""
        sel = deltas if rows is None else deltas[rows]
        total = check_aggregation(sel, weights, params.shape)
        coef = torch.tensor([w / total for w in weights], dtype=torch.float64).pin_memory().to(
            params.device, non_blocking=True)
        fedavg_device(sel, coef, params, params)
        return params

    def correct(self, params: torch.Tensor) -> int:
        if self.n_test == 0:
            return 0
        return count_correct(self.x_test, self.y_test, params, self.n_classes)

    def accuracy(self, params: torch.Tensor) -> float:
        return 0.0 if self.n_test == 0 else self.correct(params) / self.n_test


CLIENT_DTYPE = np.dtype([("x", "<u8"), ("y", "<u8"), ("perm", "<u8"), ("n_rows", "<i4"), ("n_batches", "<i4"),
                         ("batch_size", "<i4"), ("lr", "<f4"), ("delta", "<u8")])
assert CLIENT_DTYPE.itemsize == C.sizeof(_abi.Client)


def delta_buffer(k: int, P: int, dev) -> torch.Tensor:
    """[k, P] fp32 view with a 16-byte aligned row stride (vectorised FedAvg loads)."""
    ld = (P + 3) // 4 * 4
    return torch.empty((k, ld), dtype=torch.float32, device=dev)[:, :P]


def run_experiment(cfg: FleetConfig, fleet: list[ClientProfile], data: DataParams | None = None,
                   train: TrainParams | None = None, trace: list[dict] | None = None) -> ExperimentReport:
    """cfg.rounds seeded rounds: selection -> native DES -> batched GPU training -> FedAvg -> accuracy."""
    cfg.validate(fleet_size=len(fleet))
    if cfg.rounds < 1:
        raise ConfigError("rounds must be >= 1")
    data = data or DataParams()
    train = train or TrainParams(enabled=False)
    by_id = {p.client_id: p for p in fleet}
    if len(by_id) != len(fleet):
        raise ConfigError("duplicate client ids in fleet")
    ids = sorted(by_id)
    selector = random.Random(f"{cfg.seed}:selection")
    sim = RoundSimulator(by_id)

    fed = params = None
    if train.enabled:
        n_total = sum(p.workload.num_samples for p in fleet)
        # fl_core.py:41-115's dataset + partition, generated in HBM bit for bit (devicedata.reference_federation)
        fed = reference_federation([(p.client_id, p.workload.num_samples) for p in fleet], data.features,
                                   data.classes, max(math.ceil(n_total / 0.8), 10), stable_seed("data", cfg.seed),
                                   data.alpha, stable_seed("partition", cfg.seed))
        params = torch.from_numpy(init_params(data.features, data.classes)).to(device())

    report = ExperimentReport()
    now = 0.0
    if fed is not None and trace is None:
        # the serving path: pipelined planning + one launch per kernel per round
        runner = FederatedRunner(fed, by_id, cfg, train.lr, params=params)

        def record(plan, acc):
            report.rounds.append(plan.report.full() if hasattr(plan.report, "full") else plan.report)
            report.participants.append(list(plan.all_participants))

        report.accuracy_series.extend(runner.run(cfg.rounds, on_round=record))
        now = runner.now
        report.total_time = now
        report.final_params = params.cpu().numpy()
        return report
    for r in range(cfg.rounds):
        who = selector.sample(ids, cfg.participants_per_round)
        rep, seg = sim.run(who, cfg, t0=now, round_index=r, want_trace=trace is not None)
        if trace is not None:
            trace.extend(seg)
        report.rounds.append(rep)
        report.participants.append(list(who))
        round_end = now + rep.makespan
        if fed is not None:
            workloads = [by_id[c].workload for c in who]
            seeds = [stable_seed("train", cfg.seed, r, c) for c in who]
            deltas = fed.train(params, who, workloads, train.lr, seeds)
            weights = [float(w.num_samples) for w in workloads]
            if cfg.aggregation == "sync":
                fed.aggregate(params, deltas, weights)
                report.accuracy_series.append((round_end, fed.accuracy(params)))
            else:
                ends = [rep.per_client_end[c] for c in who]
                order = sorted(range(len(who)), key=lambda i: (ends[i], who[i]))
                for k in range(0, len(order), cfg.async_buffer):
                    chunk = order[k:k + cfg.async_buffer]
                    fed.aggregate(params, deltas, [weights[i] for i in chunk], rows=chunk)
                    report.accuracy_series.append((ends[chunk[-1]], fed.accuracy(params)))
        now = round_end
    report.total_time = now
    report.final_params = params.cpu().numpy() if params is not None else None
    return report


# ---------------------------------------------------------------------------------------------
# Pipelined round execution (the serving path)
# ---------------------------------------------------------------------------------------------


@dataclass
class RoundPlan:
    """Everything the host decides for one round before the GPU runs it."""

    round_index: int
    participants: list[str]          # this rank's participants, selection order
    all_participants: list[str]      # the whole round's selection (all ranks)
    report: RoundReport
    t0: float
    weights: list[float]             # this rank's float(num_samples)
    coef: np.ndarray                 # this rank's w_i / W (W over all ranks)
    slot: int                        # pinned / device plan buffer used
    perm_words: int
    desc: np.ndarray                 # CLIENT_DTYPE records (delta + perm pointers filled)
    meta_bytes: int = 0              # device-plan mode: packed (seed, rows, perms, offset) bytes
    max_rows: int = 0
    plan_launched: bool = False      # its [H2D + permutations] graph is already queued
    chunks: list | None = None       # async: [(end time, local delta rows, coefficients)] in (end, id) order


class FederatedRunner:
    """Round-after-round FedHC execution with host planning overlapped with the GPU.

    plan(r)   [host, planner thread]  selection -> native DES -> native seeds ->
              native PCG64 permutations straight into a pinned slot -> descriptors
    launch(p) [host -> GPU, one stream]  H2D of the plan, fedhc_local_train (all
              participants), fedhc_fedavg (partial + NCCL all-reduce when sharded),
              fedhc_eval; the accuracy count is copied D2H into the slot's pinned word.
    run()     a bounded pipeline: the planner thread runs up to two rounds ahead
              (3 plan slots recycled through a free-slot queue, each guarded by the
              CUDA event of its H2D copy), and the main thread launches round r+1
              before reading round r's accuracy, so the GPU always has the next
              round queued.  Every round still copies its inputs H2D and reads its
              result D2H.

    Sync FedAvg semantics (engine.py:350-353); `world`/`rank` shard participants
    (weak scaling, one all-reduce of fp64 partial sums per round).
    """

    SLOTS = 3

    def __init__(self, fed: DeviceFederation, fleet: dict[str, ClientProfile], cfg: FleetConfig, lr: float,
                 params: torch.Tensor | None = None, world: int = 1, rank: int = 0, group=None,
                 plan_threads: int = 0, device_permutations: bool = True, use_graphs: bool = False,
                 green_side: bool = True, test_sharded: bool = False, native: bool = True):
        from .sharding import shard_bounds

        self.fed, self.cfg, self.lr = fed, cfg, float(lr)
        # engine.py:354-364: async aggregation applies the round's deltas in chunks of async_buffer
        self.async_buffer = int(cfg.async_buffer) if cfg.aggregation == "async" else 0
        self.by_id = fleet
        self.ids = sorted(fleet)
        self.sim = RoundSimulator(fleet)
        self.world, self.rank, self.group = world, rank, group
        self._shard_bounds = shard_bounds
        self.selector = random.Random(f"{cfg.seed}:selection")
        # accuracy (fl_core.py:154-160): every rank counts a slice of the test rows, one int64 all-reduce.
        # test_sharded=True: `fed` already holds only this rank's slice (run() then needs n_test_total);
        # otherwise the runner takes its shard_bounds slice of the full test set itself.
        self.test_sharded = bool(test_sharded)
        if world > 1 and not test_sharded:
            tlo, thi = shard_bounds(fed.n_test, world, rank)
            self._xt, self._yt, self._nt = fed.x_test[tlo:thi], fed.y_test[tlo:thi], thi - tlo
        else:
            self._xt, self._yt, self._nt = fed.x_test, fed.y_test, fed.n_test
        dev = fed.x.device
        self.dev = dev
        self.params = params if params is not None else torch.zeros(fed.P, dtype=torch.float64, device=dev)
        # LPT may give a rank more than ceil(n / world) light clients: size the buffers for the worst case
        k_max = max(cfg.participants_per_round, 1)
        self.deltas = delta_buffer(k_max, fed.P, dev)
        self.partial = torch.empty(fed.P, dtype=torch.float64, device=dev)
        self.one = torch.ones(1, dtype=torch.float64, device=dev)
        self._repr = {cid: repr(cid).encode() for cid in self.ids}
        # per-round host work in plain arrays: repr pointers for the native seed hash, simulator indices,
        # the one-time budget > theta screen (such participants take sim.run's error path)
        self._repr_keep = [C.c_char_p(self._repr[c]) for c in self.ids]
        self._repr_ptr = np.array([C.cast(b, C.c_void_p).value for b in self._repr_keep], dtype=np.uint64)
        self._sim_idx = np.array([self.sim.index[c] for c in self.ids], dtype=np.int32)
        self._over_theta = np.array([fleet[c].resource_budget > cfg.theta for c in self.ids], dtype=bool)
        n = self.SLOTS
        self._cap = [0] * n
        self._pinned = [None] * n
        self._dev_plan = [None] * n
        self._plan_done = [None] * n   # event: H2D of the slot's plan finished
        nb = k_max * CLIENT_DTYPE.itemsize
        self._desc_dev = [torch.empty(nb, dtype=torch.uint8, device=dev) for _ in range(n)]
        self._desc_pin = [torch.empty(nb, dtype=torch.uint8).pin_memory() for _ in range(n)]
        self._coef_pin = [torch.empty(k_max, dtype=torch.float64).pin_memory() for _ in range(n)]
        self._coef_dev = [torch.empty(k_max, dtype=torch.float64, device=dev) for _ in range(n)]
        self.correct_dev = torch.zeros(1, dtype=torch.int64, device=dev)
        self._chunk_dev = None
        self._correct_pin = [torch.zeros(1, dtype=torch.int64).pin_memory() for _ in range(n)]
        self._result_ev = [None] * n
        self.plan_threads = plan_threads
        # device-plan mode: the batch permutations are generated on the GPU (perm_kernel) on a side
        # stream; the host ships only (seed, n_rows, n_perms, offset) per client.
        self.device_permutations = device_permutations
        self._meta_pin = [torch.empty(k_max * 24, dtype=torch.uint8).pin_memory() for _ in range(n)]
        self._meta_dev = [torch.empty(k_max * 24, dtype=torch.uint8, device=dev) for _ in range(n)]
        self._plan_stream = torch.cuda.Stream(device=dev)
        # Side-work SM partition (green_side, single GPU): the one-CTA-per-client train kernel needs k_max SMs
        # with all their shared memory and registers, so a batch-order (perm_kernel) or accuracy CTA resident
        # on an SM when the next round's training launches makes a train CTA wait for it (measured: those
        # rounds took 2x).  Both side streams live in green contexts confined to the SM groups the training
        # does not need -- the permutations on one window, the accuracy on another (they overlap each other
        # and the training).  The train kernel stays in the primary context.  Falls back to ordinary streams
        # without green-context support or without spare SM groups.
        self._green = None
        self._eval_ctas = None
        # FEDHC_NO_GREEN_SIDE=1: ordinary side streams (ncu cannot replay kernels launched into green contexts)
        if green_side and world == 1 and not os.environ.get("FEDHC_NO_GREEN_SIDE"):
            try:
                from .live import GreenPartitions
                gp = GreenPartitions(dev.index if dev.index is not None else 0)
                # groups the training needs: one SM per client for the one-CTA trainers; the cluster trainers
                # (62 classes, F > 784) fill the GPU, so no window is spare and side work shares the device
                spc = train_sms_per_client(fed.n_features, fed.n_classes)
                need = -(-k_max * spc // gp.sms_per_group)
                spare = gp.n_groups - need
                if spare >= 1:
                    # permutations: the SMs outside every group (28 of 148 on a B200: ~0.4 ms for 100 clients
                    # of 6400 rows); accuracy: the spare groups (2 x 8 SMs)
                    eval_first, eval_n = need, spare
                    if device_permutations:
                        try:
                            raw, _ = gp.stream_rest(need, 0)
                        except ValueError:  # every SM is in a group: give the permutations one spare group
                            if spare < 2:
                                raise
                            raw = gp.stream(need, 1)
                            eval_first, eval_n = need + 1, spare - 1
                        self._plan_stream = torch.cuda.ExternalStream(raw, device=dev)
                    self._eval_stream_raw = gp.stream(eval_first, eval_n)
                    self._eval_ctas = eval_n * gp.sms_per_group  # one CTA per SM of the window
                    self._green = gp
            except Exception:  # no green-context support in this driver: keep the ordinary streams
                self._green = None
        self._train_done = [None] * n   # event: the slot's train kernel retired (plan buffer reusable)
        # one pinned / device staging block per slot for the device-plan mode: [meta 24k | desc | coef 8k],
        # copied H2D in one transfer on the plan stream
        self._stage_pin = [torch.empty(k_max * (24 + CLIENT_DTYPE.itemsize + 8), dtype=torch.uint8).pin_memory()
                           for _ in range(n)]
        self._stage_dev = [torch.empty(k_max * (24 + CLIENT_DTYPE.itemsize + 8), dtype=torch.uint8, device=dev)
                           for _ in range(n)]
        self._ev_plan = [torch.cuda.Event() for _ in range(n)]
        self._ev_train = [torch.cuda.Event() for _ in range(n)]
        self._ev_result = [torch.cuda.Event() for _ in range(n)]
        # single-GPU eager rounds: accuracy of round r runs on its own stream, overlapping round r + 1's
        # training (both only read the params); round r + 1's FedAvg waits for it before writing them
        self._eval_stream = (torch.cuda.ExternalStream(self._eval_stream_raw, device=dev) if self._green is not None
                             else torch.cuda.Stream(device=dev))
        self._sms = torch.cuda.get_device_properties(dev).multi_processor_count
        self._ev_agg = [torch.cuda.Event() for _ in range(n)]
        self._eval_done = None
        # per-client constants, indexed like self.ids (vectorised planning)
        F = fed.n_features
        off = np.array([fed.offset[c][0] for c in self.ids], np.int64)
        self._c_rows = np.array([fed.offset[c][1] for c in self.ids], np.int64)
        ns = np.array([fleet[c].workload.num_samples for c in self.ids], np.int64)
        bs = np.array([fleet[c].workload.batch_size for c in self.ids], np.int64)
        self._c_w = ns.astype(np.float64)
        from .sharding import client_cost, lpt_shards
        self._lpt = lpt_shards
        self._c_cost = np.array([client_cost(n, b, rws) for n, b, rws in zip(ns, bs, self._c_rows)], np.float64)
        self._c_bs = bs
        self._c_steps = -(-ns // bs)
        per_epoch = -(-self._c_rows // bs)
        self._c_nperm = np.where(self._c_rows == 0, 0,
                                 np.maximum(1, -(-self._c_steps // np.maximum(per_epoch, 1))))
        self._rows_max = int(self._c_rows.max()) if len(self._c_rows) else 0
        self._bs_max = int(bs.max()) if len(bs) else 1
        # CUDA graphs per slot (world == 1, device plans): [H2D + permutations] on the plan stream and
        # [train + FedAvg + eval + D2H] on the main stream, each replayed with one launch per round
        self.use_graphs = use_graphs and device_permutations and world == 1
        self._graphs = [None] * n
        self._cap_stream = torch.cuda.Stream(device=dev)
        self._c_xptr = np.ascontiguousarray((fed.x.data_ptr() + off * (F * 4)).astype(np.uint64))
        self._c_yptr = np.ascontiguousarray((fed.y.data_ptr() + off * 4).astype(np.uint64))
        self._c_rows32 = self._c_rows.astype(np.int32)
        self._c_nperm32 = self._c_nperm.astype(np.int32)
        self._c_steps32 = self._c_steps.astype(np.int32)
        self._c_bs32 = self._c_bs.astype(np.int32)
        # the selector's MT19937 state (Random.getstate(): 624 words + index) for the native sample
        self._mt = np.array(self.selector.getstate()[1], dtype=np.uint32)
        self._who_buf = np.zeros(max(cfg.participants_per_round, 1), dtype=np.int32)
        self.now = 0.0
        self.round = 0
        self._prefetch = None  # next run()'s first RoundPlan, planned during the previous run
        self.h2d_bytes = 0
        self.d2h_bytes = 8
        self.host_s = {"select+des": 0.0, "seeds": 0.0, "permutations": 0.0, "descriptors": 0.0, "launch": 0.0}
        # native round loop (single GPU, device batch order, eager launches): plan / launch / result are one
        # GIL-free libfedhc call each (fedhc_runner_*); the Python path below stays for world > 1 and graphs
        self._native = None
        if native and world == 1 and device_permutations and not self.use_graphs:
            self._native_init(k_max)

    def _native_init(self, k_max: int) -> None:
        fed, cfg, n = self.fed, self.cfg, self.SLOTS
        dev = self.dev
        kp = cfg.participants_per_round
        # plan buffers sized for the kp largest shards (no reallocation inside the loop)
        words = np.sort(self._c_rows * self._c_nperm)[::-1][:kp].sum() if kp else 0
        cap = max(int(words), 1)
        self._n_plan = [torch.empty(cap, dtype=torch.int32, device=dev) for _ in range(n)]
        blk = max(kp, 1) * (24 + CLIENT_DTYPE.itemsize + 8)
        self._n_stage_pin = [torch.empty(blk, dtype=torch.uint8).pin_memory() for _ in range(n)]
        self._n_stage_dev = [torch.empty(blk, dtype=torch.uint8, device=dev) for _ in range(n)]
        kq = max(kp, 1)
        self._n_correct_dev = torch.zeros(n * kq, dtype=torch.int64, device=dev)
        self._n_correct_pin = torch.zeros(n * kq, dtype=torch.int64).pin_memory()
        if self.async_buffer:
            self._n_async_pin = [torch.empty(16 * kq, dtype=torch.uint8).pin_memory() for _ in range(n)]
            self._n_async_dev = [torch.empty(16 * kq, dtype=torch.uint8, device=dev) for _ in range(n)]
            self._n_snap = [torch.empty(kq * fed.P, dtype=torch.float64, device=dev) for _ in range(n)]
        else:
            self._n_async_pin = self._n_async_dev = self._n_snap = []
        ptrs = lambda ts: np.array([t.data_ptr() for t in ts], dtype=np.uint64)  # noqa: E731
        self._n_keep = [ptrs(self._n_stage_pin), ptrs(self._n_stage_dev), ptrs(self._n_plan),
                        np.ascontiguousarray(self._over_theta.astype(np.uint8)),
                        np.ascontiguousarray(self._sim_idx.astype(np.int32)), np.ascontiguousarray(self._c_w),
                        ptrs(self._n_async_pin), ptrs(self._n_async_dev), ptrs(self._n_snap)]
        sp, sd, pd, ot, si, w, ah, ad, sn = self._n_keep
        sim = self.sim
        des = _abi.DesConfig(float(cfg.theta), int(cfg.max_executors), 0 if cfg.scheduler_kind == "resource-aware"
                             else 1, int(bool(cfg.dynamic_parallelism)), float(cfg.alpha), float(cfg.beta),
                             float(cfg.launch_latency), float(cfg.terminate_latency), float(cfg.upload_latency))
        if cfg.scheduler_kind not in ("resource-aware", "greedy"):
            raise KeyError(cfg.scheduler_kind)
        xs = fed.x_split
        c = _abi.RunnerConfig()
        c.reprs, c.rows, c.n_perms = self._repr_ptr.ctypes.data, self._c_rows32.ctypes.data, self._c_nperm32.ctypes.data
        c.n_batches, c.batch_size = self._c_steps32.ctypes.data, self._c_bs32.ctypes.data
        c.xptr, c.yptr, c.weight = self._c_xptr.ctypes.data, self._c_yptr.ctypes.data, w.ctypes.data
        c.over_theta, c.sim_index, c.mt_state = ot.ctypes.data, si.ctypes.data, self._mt.ctypes.data
        c.sim = sim._sim
        c.des_clients = C.cast(sim._clients, C.c_void_p).value
        c.des_ids = C.cast(sim._id_arr, C.c_void_p).value
        c.params, c.deltas = self.params.data_ptr(), self.deltas.data_ptr()
        c.delta_stride_bytes = self.deltas.stride(0) * 4
        c.split_offset = (xs.data_ptr() - fed.x.data_ptr()) if xs is not None else 0
        c.x_test, c.y_test, c.n_test = self._xt.data_ptr(), self._yt.data_ptr(), int(self._nt)
        c.correct_dev, c.correct_host = self._n_correct_dev.data_ptr(), self._n_correct_pin.data_ptr()
        c.stage_host, c.stage_dev, c.plan_dev = sp.ctypes.data, sd.ctypes.data, pd.ctypes.data
        c.plan_cap_words = cap
        c.plan_stream, c.eval_stream = self._plan_stream.cuda_stream, self._eval_stream.cuda_stream
        c.seed, c.des_cfg, c.lr = int(cfg.seed), des, self.lr
        if self.async_buffer:
            c.async_host, c.async_dev, c.snapshots = ah.ctypes.data, ad.ctypes.data, sn.ctypes.data
        c.async_buffer = self.async_buffer
        c.n_fleet, c.participants, c.slots = len(self.ids), kp, n
        c.n_features, c.n_classes, c.max_batch = fed.n_features, fed.n_classes, self._bs_max
        c.split = 1 if xs is not None else 0
        c.eval_ctas = self._eval_ctas if self._eval_ctas is not None else self._side_ctas(kp)
        c.rows_max = self._rows_max
        self._n_cfg = c
        h = C.c_void_p()
        _abi.check(_abi.lib.fedhc_runner_create(C.byref(c), C.byref(h)))
        self._native = h
        # per-slot host outputs of fedhc_runner_plan
        kq = max(kp, 1)
        self._n_out = []
        for _ in range(n):
            o = {"selected": np.zeros(kq, np.int32), "starts": np.zeros(kq), "ends": np.zeros(kq),
                 "launch": np.zeros(kq, np.int32), "upload": np.zeros(kq, np.int32),
                 "par_t": np.zeros(4 * kq + 16), "par_n": np.zeros(4 * kq + 16, np.int32),
                 "chunk_end": np.zeros(kq), "counts": np.zeros(kq, np.int64)}
            info = _abi.RunnerPlanInfo()
            info.selected, info.starts, info.ends = (o["selected"].ctypes.data, o["starts"].ctypes.data,
                                                     o["ends"].ctypes.data)
            info.launch_order, info.upload_order = o["launch"].ctypes.data, o["upload"].ctypes.data
            info.par_t, info.par_n, info.par_cap = o["par_t"].ctypes.data, o["par_n"].ctypes.data, 4 * kq + 16
            info.chunk_end = o["chunk_end"].ctypes.data
            o["info"] = info
            self._n_out.append(o)

    def __del__(self):
        h = getattr(self, "_native", None)
        if h:
            _abi.lib.fedhc_runner_destroy(h)
            self._native = None

    def _native_plan(self, r: int, t0: float, slot: int) -> RoundPlan:
        """fedhc_runner_plan (selection, DES, packing, H2D + device batch order) -> RoundPlan."""
        tick = time.perf_counter()
        o = self._n_out[slot]
        info = o["info"]
        _abi.check(_abi.lib.fedhc_runner_plan(self._native, int(r), float(t0), slot, C.byref(info)))
        kp = self.cfg.participants_per_round
        who = [self.ids[i] for i in o["selected"][:kp].tolist()]
        if info.over_theta:  # the reference's ConfigError, from the same selection
            self.sim.run(who, self.cfg, t0=t0, round_index=r, want_trace=False)
        npar = info.n_par
        if npar < 0:
            raise RuntimeError("runner: parallelism timeline buffer too small")
        rep = LeanRoundReport(r, info.makespan, info.utilization, info.vacancy_area, info.throughput,
                              bool(info.degenerate), who, o["launch"][:info.n_launched].copy(),
                              o["upload"][:info.n_uploaded].copy(), o["starts"][:kp].copy(), o["ends"][:kp].copy(),
                              o["par_t"][:npar].copy() if npar else None,
                              o["par_n"][:npar].copy() if npar else None, self.sim.budget)
        self.h2d_bytes = int(info.h2d_bytes)
        self.host_s["select+des"] += time.perf_counter() - tick
        chunks = [(float(t), None, None) for t in o["chunk_end"][:info.n_chunks]] if self.async_buffer else None
        return RoundPlan(r, who, who, rep, t0, [], np.zeros(0), slot, int(info.perm_words), None,
                         24 * kp, int(info.max_rows), plan_launched=True, chunks=chunks)

    def _native_run(self, rounds: int, n_test: int, on_round) -> list:
        """run() on the native loop: a planner thread (fedhc_runner_plan) feeding the launching thread."""
        import queue
        import threading

        ready: queue.Queue = queue.Queue(maxsize=self.SLOTS - 1)
        free: queue.Queue = queue.Queue()
        for sl in range(self.SLOTS):
            free.put(sl)
        failure = []
        t_start, r0 = self.now, self.round

        def planner():
            t = t_start
            try:
                torch.cuda.set_device(self.dev)
                for i in range(rounds):
                    pl = self._native_plan(r0 + i, t, free.get())
                    t = pl.t0 + pl.report.makespan
                    ready.put(pl)
            except BaseException as exc:  # surface planner errors in the caller
                failure.append(exc)
                ready.put(None)

        th = threading.Thread(target=planner, daemon=True)
        th.start()
        series, pending = [], None
        hs = self.host_s
        stream = torch.cuda.current_stream().cuda_stream
        last = [None]
        try:
            for _ in range(rounds):
                t0 = time.perf_counter()
                p = ready.get()
                hs["wait_plan"] = hs.get("wait_plan", 0.0) + time.perf_counter() - t0
                if p is None:
                    raise failure[0]
                t1 = time.perf_counter()
                _abi.check(_abi.lib.fedhc_runner_launch(self._native, p.slot, stream))
                hs["launch"] += time.perf_counter() - t1
                if pending is not None:
                    t0 = time.perf_counter()
                    series.extend(self._native_finish(pending, n_test, on_round))
                    free.put(pending.slot)
                    hs["wait_gpu"] = hs.get("wait_gpu", 0.0) + time.perf_counter() - t0
                last[0] = p
                pending = p
            series.extend(self._native_finish(pending, n_test, on_round))
            free.put(pending.slot)
        finally:
            th.join()
        self.round += rounds
        self.now = last[0].t0 + last[0].report.makespan
        return series

    def _native_finish(self, p: RoundPlan, n_test: int, on_round) -> list:
        counts = self._n_out[p.slot]["counts"]
        _abi.check(_abi.lib.fedhc_runner_result(self._native, p.slot, counts.ctypes.data))
        return self._series_entries(p, counts, n_test, on_round)

    def _series_entries(self, p: RoundPlan, counts, n_test: int, on_round) -> list:
        """[(time, accuracy)] of a finished round: one entry (sync) or one per aggregation chunk (async)."""
        if p.chunks is None:
            acc = int(counts[0]) / n_test if n_test else 0.0
            out = [(p.t0 + p.report.makespan, acc)]
        else:
            out = [(t, int(counts[i]) / n_test if n_test else 0.0) for i, (t, _, _) in enumerate(p.chunks)]
        if on_round is not None:
            on_round(p, out[-1][1])
        return out

    # ---- host side ---------------------------------------------------------
    def _ensure(self, slot: int, words: int):
        if self._plan_done[slot] is not None:
            self._plan_done[slot].synchronize()   # the GPU finished copying this slot's previous plan
        if words > self._cap[slot]:
            cap = max(words, 2 * self._cap[slot])
            self._cap[slot] = cap
            self._pinned[slot] = torch.empty(cap, dtype=torch.int32).pin_memory()
            self._dev_plan[slot] = torch.empty(cap, dtype=torch.int32, device=self.dev)

    def plan(self, r: int, t0: float, slot: int | None = None) -> RoundPlan:
        cfg = self.cfg
        slot = (r % self.SLOTS) if slot is None else slot
        tick = time.perf_counter()
        # random.sample draws indices from len(population) only: sampling range(n) is the same draw
        # sequence as sampling the ids (engine.py:327), and gives the fleet indices directly.  Native:
        # CPython's sample on the selector's MT19937 state (fedhc_mt_sample), bit-exact.
        kp = cfg.participants_per_round
        wi32 = self._who_buf[:max(kp, 1)]
        _abi.check(_abi.lib.fedhc_mt_sample(self._mt.ctypes.data, len(self.ids), kp, wi32.ctypes.data))
        wi = wi32[:kp].astype(np.int64)
        who = [self.ids[i] for i in wi.tolist()]
        if self._over_theta[wi].any():   # sim.run raises the reference's ConfigError
            rep, _ = self.sim.run(who, cfg, t0=t0, round_index=r, want_trace=False)
        else:
            rep = self.sim.run_lean(self._sim_idx[wi], who, cfg, t0=t0, round_index=r)
        t1 = time.perf_counter()
        if self.world > 1:   # LPT over the GPU cost (rows processed) of each participant
            sel = self._lpt(self._c_cost[wi].tolist(), self.world)[self.rank]
        else:
            sel = list(range(len(who)))
        mine = [who[j] for j in sel]
        mi = wi[sel] if sel else np.zeros(0, np.int64)
        k = len(mine)
        w_all = np.ascontiguousarray(self._c_w[wi])
        total = _abi.lib.fedhc_py_float_sum(w_all.ctypes.data, kp)  # CPython 3.12 float sum(), as the reference
        # fl_core.fedavg's validation (fl_core.py:201-212), raised before any device work: the reference
        # raises it at the round's FedAvg (engine.py:351), after a round that trains nothing useful
        if not who:
            raise AggregationError("no deltas to aggregate")
        if total == 0:
            raise AggregationError("weights must not all be zero")
        my_w = w_all[sel].tolist()
        chunks = self._async_chunks(rep, who, w_all, sel) if self.async_buffer else None
        if self.device_permutations:
            p = self._plan_packed(r, t0, slot, rep, who, mine, mi, my_w, total, tick, t1)
            p.chunks = chunks
            return p
        coef = np.asarray(my_w, np.float64) / total
        reprs = self._repr_ptr[mi] if k else self._repr_ptr[:1]   # const char* per participant
        train_seeds = np.zeros(max(k, 1), np.uint64)
        rng_seeds = np.zeros(max(k, 1), np.uint64)
        _abi.check(_abi.lib.fedhc_round_seeds(int(cfg.seed), int(r), reprs.ctypes.data_as(C.POINTER(C.c_char_p)), k,
                                              train_seeds.ctypes.data, rng_seeds.ctypes.data))
        t2 = time.perf_counter()
        rows = self._c_rows[mi]
        perms = self._c_nperm[mi]
        sizes = rows * perms
        offs = np.zeros(k, np.int64)
        if k > 1:
            np.cumsum(sizes[:-1], out=offs[1:])
        at = int(sizes.sum()) if k else 0
        self._ensure(slot, max(at, 1))
        meta_bytes = 0
        if at and self.device_permutations:
            buf = self._stage_pin[slot].numpy()
            buf[:8 * k] = rng_seeds[:k].view(np.uint8)
            buf[8 * k:12 * k] = rows.astype(np.int32).view(np.uint8)
            buf[12 * k:16 * k] = perms.astype(np.int32).view(np.uint8)
            buf[16 * k:24 * k] = offs.view(np.uint8)
            meta_bytes = 24 * k
            self._stage_pin[slot].numpy()[meta_bytes + k * CLIENT_DTYPE.itemsize:][:8 * k] = coef.view(np.uint8)
        elif at:
            native_permutations(rng_seeds[:k], rows.tolist(), perms.tolist(), out=self._pinned[slot].numpy(),
                                threads=self.plan_threads)
        t3 = time.perf_counter()
        desc = np.zeros(k, dtype=CLIENT_DTYPE)
        if k:
            desc["x"] = self._c_xptr[mi]
            desc["y"] = self._c_yptr[mi]
            desc["perm"] = self._dev_plan[slot].data_ptr() + offs * 4
            desc["n_rows"] = rows
            desc["n_batches"] = self._c_steps[mi]
            desc["batch_size"] = self._c_bs[mi]
            desc["lr"] = self.lr
            desc["delta"] = self.deltas.data_ptr() + np.arange(k, dtype=np.int64) * (self.deltas.stride(0) * 4)
            if meta_bytes:  # device-plan staging block [meta | descriptors | coefficients] complete
                self._stage_pin[slot].numpy()[meta_bytes:meta_bytes + k * CLIENT_DTYPE.itemsize] = desc.view(np.uint8)
        t4 = time.perf_counter()
        hs = self.host_s
        hs["select+des"] += t1 - tick
        hs["seeds"] += t2 - t1
        hs["permutations"] += t3 - t2
        hs["descriptors"] += t4 - t3
        return RoundPlan(r, mine, who, rep, t0, my_w, coef, slot, at, desc, meta_bytes,
                         int(rows.max()) if k else 0, chunks=chunks)

    def _async_chunks(self, rep, who, w_all, sel) -> list:
        """engine.py:355-364: the round's participants in (per_client_end, id) order, chunks of async_buffer;
        per chunk (end of its last client, this rank's delta rows, their w_i / W_chunk)."""
        ends = rep.end_times() if hasattr(rep, "end_times") else np.array([rep.per_client_end[c] for c in who])
        order = sorted(range(len(who)), key=lambda i: (ends[i], who[i]))
        local = {g: j for j, g in enumerate(sel)}
        w = w_all.tolist()
        out = []
        for at in range(0, len(order), self.async_buffer):
            ch = order[at:at + self.async_buffer]
            wc = float(sum(w[i] for i in ch))  # fl_core.fedavg's total over the chunk (CPython float sum)
            if wc == 0:
                raise AggregationError("weights must not all be zero")
            mine = [i for i in ch if i in local]
            out.append((float(ends[ch[-1]]), [local[i] for i in mine], [w[i] / wc for i in mine]))
        return out

    def _plan_packed(self, r, t0, slot, rep, who, mine, mi, my_w, total, tick, t1) -> RoundPlan:
        """Device batch order: seeds, the [meta | descriptors | coefficients] staging block and the plan
        buffer in one native call (fedhc_round_pack, GIL released)."""
        k = len(mine)
        at = int((self._c_rows[mi] * self._c_nperm[mi]).sum()) if k else 0
        self._ensure(slot, max(at, 1))
        pin = self._stage_pin[slot]
        words, mrows = C.c_int64(), C.c_int32()
        mi64 = np.ascontiguousarray(mi, dtype=np.int64)
        _abi.check(_abi.lib.fedhc_round_pack(int(self.cfg.seed), int(r), k, mi64.ctypes.data,
                                             self._repr_ptr.ctypes.data, self._c_rows32.ctypes.data,
                                             self._c_nperm32.ctypes.data, self._c_steps32.ctypes.data,
                                             self._c_bs32.ctypes.data, self._c_xptr.ctypes.data,
                                             self._c_yptr.ctypes.data, self._c_w.ctypes.data, float(total),
                                             float(self.lr), self._dev_plan[slot].data_ptr(), self.deltas.data_ptr(),
                                             self.deltas.stride(0) * 4, pin.data_ptr(), C.byref(words),
                                             C.byref(mrows)))
        buf = pin.numpy()
        nb = k * CLIENT_DTYPE.itemsize
        meta_bytes = 24 * k if at else 0
        desc = buf[24 * k:24 * k + nb].view(CLIENT_DTYPE)
        coef = buf[24 * k + nb:24 * k + nb + 8 * k].view(np.float64)
        if not at:  # every shard empty: no device permutations (zero deltas), descriptors still launch
            desc, coef = desc.copy(), coef.copy()
        t4 = time.perf_counter()
        hs = self.host_s
        hs["select+des"] += t1 - tick
        hs["seeds"] += 0.0
        hs["permutations"] += 0.0
        hs["descriptors"] += t4 - t1
        return RoundPlan(r, mine, who, rep, t0, my_w, coef, slot, at, desc, meta_bytes, int(mrows.value))

    # ---- device side -------------------------------------------------------
    def _graph_key(self, p: RoundPlan):
        return (len(p.participants), p.meta_bytes, self._dev_plan[p.slot].data_ptr())

    def _capture(self, p: RoundPlan):
        """Capture the slot's two graphs (no execution); replayed from the next use of the slot on."""
        k, slot, mb = len(p.participants), p.slot, p.meta_bytes
        nb = k * CLIENT_DTYPE.itemsize
        tot = mb + nb + 8 * k
        dev = self._stage_dev[slot]
        md = dev.data_ptr()
        coef_t = dev[mb + nb:mb + nb + 8 * k].view(torch.float64)
        gp, gr = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.graph(gp, stream=self._cap_stream, capture_error_mode="thread_local"):
            dev[:tot].copy_(self._stage_pin[slot][:tot], non_blocking=True)
            _abi.check(_abi.lib.fedhc_batch_permutations_device(md, md + 8 * k, md + 12 * k, md + 16 * k, k,
                                                                self._dev_plan[slot].data_ptr(), self._rows_max,
                                                                stream_ptr()))
        with torch.cuda.graph(gr, stream=self._cap_stream, capture_error_mode="thread_local"):
            self.fed.launch_train(md + mb, k, self.params, self._bs_max)
            fedavg_device(self.deltas[:k], coef_t, self.params, self.params)
            self.correct_dev.zero_()
            if self._nt:
                _abi.check(_abi.lib.fedhc_eval(self._xt.data_ptr(), self._yt.data_ptr(),
                                               self._nt, self.fed.n_features, self.fed.n_classes,
                                               self.params.data_ptr(), self.correct_dev.data_ptr(), stream_ptr()))
            self._correct_pin[slot].copy_(self.correct_dev, non_blocking=True)
        self._graphs[slot] = (self._graph_key(p), gp, gr)

    def _graph_ready(self, p: RoundPlan) -> bool:
        gs = self._graphs[p.slot]
        return bool(self.use_graphs and p.participants and p.meta_bytes and gs is not None
                    and gs[0] == self._graph_key(p))

    def launch_plan(self, p: RoundPlan) -> None:
        if (self._green is not None or not self.use_graphs) and not p.plan_launched and p.meta_bytes \
                and p.participants:
            # eager, from the planner thread as soon as the round is planned: the batch order is generated
            # while earlier rounds train, off the next train kernel's critical path (on the green-context
            # stream, if any, the kernel is confined to the spare SM groups)
            k, slot, mb = len(p.participants), p.slot, p.meta_bytes
            tot = mb + k * CLIENT_DTYPE.itemsize + 8 * k
            ps = self._plan_stream
            dev = self._stage_dev[slot]
            md = dev.data_ptr()
            with torch.cuda.stream(ps):
                ps.wait_event(self._ev_train[slot])  # the slot's previous train kernel is done with its buffers
                dev[:tot].copy_(self._stage_pin[slot][:tot], non_blocking=True)
                _abi.check(_abi.lib.fedhc_batch_permutations_device(md, md + 8 * k, md + 12 * k, md + 16 * k, k,
                                                                    self._dev_plan[slot].data_ptr(), self._rows_max,
                                                                    ps.cuda_stream))
                self._ev_plan[slot].record(ps)
            p.plan_launched = True
            return
        self._launch_plan_graph(p)

    def _launch_plan_graph(self, p: RoundPlan) -> None:
        """Queue the round's [H2D + device permutations] graph on the plan stream (no-op without graphs).

        The planner thread calls this as soon as a round is planned, so its permutations are generated
        on the SMs the running round leaves idle."""
        if p.plan_launched or not self._graph_ready(p):
            return
        ps = self._plan_stream
        with torch.cuda.stream(ps):
            self._graphs[p.slot][1].replay()
            self._ev_plan[p.slot].record(ps)
        p.plan_launched = True

    def launch(self, p: RoundPlan) -> None:
        """Enqueue the round on the current stream (asynchronous); result lands in slot p.slot."""
        from .sharding import all_reduce_count, combine_partials

        tick = time.perf_counter()
        k = len(p.participants)
        slot = p.slot
        main = torch.cuda.current_stream()
        nb = k * CLIENT_DTYPE.itemsize
        if self._graph_ready(p):
            if not p.plan_launched:
                self.launch_plan(p)
            gs = self._graphs[slot]
            main.wait_event(self._ev_plan[slot])
            if self._eval_done is not None:  # an eager round's accuracy may still be reading the params
                main.wait_event(self._eval_done)
                self._eval_done = None
            self._plan_done[slot] = self._ev_plan[slot]
            gs[2].replay()
            self._ev_train[slot].record()
            self._train_done[slot] = self._ev_train[slot]
            self._ev_result[slot].record()
            self._result_ev[slot] = self._ev_result[slot]
            self.h2d_bytes = p.meta_bytes + nb + 8 * k
            self.host_s["launch"] += time.perf_counter() - tick
            return
        gs = self._graphs[slot]
        if p.meta_bytes:
            # one H2D transfer of [meta | descriptors | coefficients] on the plan stream, then the
            # device PCG64 permutations; the main stream waits for both
            ps = self._plan_stream
            mb = p.meta_bytes
            stage = self._stage_pin[slot].numpy()
            stage[mb:mb + nb] = p.desc.view(np.uint8)
            stage[mb + nb:mb + nb + 8 * k] = p.coef.view(np.uint8)
            tot = mb + nb + 8 * k
            dev = self._stage_dev[slot]
            md = dev.data_ptr()
            if not p.plan_launched:
                with torch.cuda.stream(ps):
                    ps.wait_event(self._ev_train[slot])      # the slot's previous train kernel is done with it
                    dev[:tot].copy_(self._stage_pin[slot][:tot], non_blocking=True)
                    _abi.check(_abi.lib.fedhc_batch_permutations_device(md, md + 8 * k, md + 12 * k, md + 16 * k,
                                                                        k, self._dev_plan[slot].data_ptr(),
                                                                        p.max_rows, ps.cuda_stream))
                    self._ev_plan[slot].record(ps)
            main.wait_event(self._ev_plan[slot])
            self._plan_done[slot] = self._ev_plan[slot]
            desc_ptr, coef_t = md + mb, dev[mb + nb:mb + nb + 8 * k].view(torch.float64)
            self.h2d_bytes = tot
        else:
            if p.perm_words:
                self._dev_plan[slot][:p.perm_words].copy_(self._pinned[slot][:p.perm_words], non_blocking=True)
            if k:
                self._desc_pin[slot].numpy()[:nb] = p.desc.view(np.uint8)
                self._desc_dev[slot][:nb].copy_(self._desc_pin[slot][:nb], non_blocking=True)
                self._coef_pin[slot].numpy()[:k] = p.coef
                self._coef_dev[slot][:k].copy_(self._coef_pin[slot][:k], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()
            self._plan_done[slot] = ev
            desc_ptr, coef_t = self._desc_dev[slot].data_ptr(), self._coef_dev[slot][:k]
            self.h2d_bytes = p.perm_words * 4 + nb + k * 8
        if k:
            max_b = int(p.desc["batch_size"].max())
            self.fed.launch_train(desc_ptr, k, self.params, max_b)
        self._ev_train[slot].record()
        self._train_done[slot] = self._ev_train[slot]
        if p.chunks is not None:
            self._launch_async(p, main)
        elif self.world == 1:
            if self._eval_done is not None:
                main.wait_event(self._eval_done)  # the previous round's accuracy is done reading the params
            if k:
                fedavg_device(self.deltas[:k], coef_t, self.params, self.params)
        else:
            if k:
                fedavg_device(self.deltas[:k], coef_t, None, self.partial)
            else:
                self.partial.zero_()
            combine_partials(self.partial, self.params,
                             lambda s, prm: fedavg_device(s.view(1, -1), self.one, prm, prm), self.group)
        if p.chunks is not None:
            pass  # accuracy per chunk: _launch_async
        elif self.world == 1:
            es = self._eval_stream
            self._ev_agg[slot].record(main)
            es.wait_event(self._ev_agg[slot])
            with torch.cuda.stream(es):
                self.correct_dev.zero_()
                if self._nt:
                    # overlaps the next round's training (one CTA per client): stay on the idle SMs
                    ctas = self._eval_ctas if self._eval_ctas is not None else self._side_ctas(k)
                    _abi.check(_abi.lib.fedhc_eval_ctas(self._xt.data_ptr(), self._yt.data_ptr(),
                                                        self._nt, self.fed.n_features, self.fed.n_classes,
                                                        self.params.data_ptr(), self.correct_dev.data_ptr(), ctas,
                                                        es.cuda_stream))
                self._correct_pin[slot].copy_(self.correct_dev, non_blocking=True)
                self._ev_result[slot].record(es)
            self._eval_done = self._ev_result[slot]
        else:
            self.correct_dev.zero_()
            if self._nt:
                _abi.check(_abi.lib.fedhc_eval(self._xt.data_ptr(), self._yt.data_ptr(),
                                               self._nt, self.fed.n_features, self.fed.n_classes,
                                               self.params.data_ptr(), self.correct_dev.data_ptr(), stream_ptr()))
            all_reduce_count(self.correct_dev, self.group)
            self._correct_pin[slot].copy_(self.correct_dev, non_blocking=True)
            self._ev_result[slot].record()
        self._result_ev[slot] = self._ev_result[slot]
        if self.use_graphs and p.chunks is None and k and p.meta_bytes and (gs is None or gs[0] != self._graph_key(p)):
            self._capture(p)
        self.host_s["launch"] += time.perf_counter() - tick

    def _side_ctas(self, k: int) -> int:
        """Accuracy CTAs without a green window: the SMs the one-CTA trainers leave idle beside k clients; the
        cluster trainers fill the GPU (the accuracy then runs between trainings), so it takes every SM."""
        if train_sms_per_client(self.fed.n_features, self.fed.n_classes) > 1:
            return self._sms
        return max(8, self._sms - k)

    def read_correct(self, slot: int) -> int:
        self._result_ev[slot].synchronize()
        return int(self._correct_pin[slot][0].item())

    def _launch_async(self, p: RoundPlan, main) -> None:
        """Async aggregation (engine.py:354-364) on the Python path: per chunk, this rank's partial FedAvg
        (pointer rows, w_i / W_chunk), one all-reduce of the fp64 partials, the apply, and the chunk's sharded
        accuracy count; one all-reduce of the round's counts and one D2H."""
        from .sharding import all_reduce_count, combine_partials
        slot, nc = p.slot, len(p.chunks)
        if self._chunk_dev is None or self._chunk_dev.shape[0] < nc:
            self._chunk_dev = torch.zeros(max(nc, 1), dtype=torch.int64, device=self.dev)
        counts = self._chunk_dev[:nc]
        counts.zero_()
        row0 = self.deltas.data_ptr()
        stride = self.deltas.stride(0) * 4
        for ci, (_, rows, coef) in enumerate(p.chunks):
            if rows:
                ptr = torch.tensor([row0 + j * stride for j in rows], dtype=torch.int64).to(self.dev, non_blocking=True)
                cf = torch.tensor(coef, dtype=torch.float64).to(self.dev, non_blocking=True)
                if self.world == 1:
                    fedavg_device(self.deltas, cf, self.params, self.params, rows=ptr)
                else:
                    fedavg_device(self.deltas, cf, None, self.partial, rows=ptr)
            elif self.world > 1:
                self.partial.zero_()
            if self.world > 1:
                combine_partials(self.partial, self.params,
                                 lambda s_, prm: fedavg_device(s_.view(1, -1), self.one, prm, prm), self.group)
            if self._nt:
                _abi.check(_abi.lib.fedhc_eval(self._xt.data_ptr(), self._yt.data_ptr(), self._nt,
                                               self.fed.n_features, self.fed.n_classes, self.params.data_ptr(),
                                               counts[ci:ci + 1].data_ptr(), stream_ptr()))
        all_reduce_count(counts, self.group)
        if self._correct_pin[slot].shape[0] < nc:
            self._correct_pin[slot] = torch.zeros(nc, dtype=torch.int64).pin_memory()
        self._correct_pin[slot][:nc].copy_(counts, non_blocking=True)
        self._ev_result[slot].record()
        self._eval_done = None

    def run(self, rounds: int, n_test_total: int | None = None, on_round=None):
        """Run `rounds` rounds; returns [(round_end_time, accuracy)] (engine.py:350-353 sync semantics)."""
        import queue
        import threading

        if n_test_total is None:
            if self.test_sharded and self.world > 1:
                raise ValueError("FederatedRunner(test_sharded=True) needs n_test_total (the global test-set size)")
            n_test_total = self.fed.n_test
        n_test = n_test_total
        if rounds <= 0:
            return []
        if self._native is not None:
            return self._native_run(rounds, n_test, on_round)
        ready: queue.Queue = queue.Queue(maxsize=self.SLOTS - 1)
        free: queue.Queue = queue.Queue()
        # the previous call planned this call's first round while its last round drained (no pipeline fill)
        pre, self._prefetch = self._prefetch, None
        for sl in range(self.SLOTS):
            if not isinstance(pre, RoundPlan) or sl != pre.slot:
                free.put(sl)
        failure = []

        def planner():
            t, r0 = self.now, self.round
            try:
                torch.cuda.set_device(self.dev)  # bind the device context in this thread (it launches plan work)
                start = 0
                if isinstance(pre, BaseException):  # planning this round failed during the previous call
                    raise pre
                if pre is not None:
                    t = pre.t0 + pre.report.makespan
                    ready.put(pre)
                    start = 1
                for i in range(start, rounds):
                    slot = free.get()
                    pl = self.plan(r0 + i, t, slot)
                    # queue the round's [H2D + device permutations] graph right away, so the batch
                    # order is generated on the SMs the running round leaves idle
                    self.launch_plan(pl)
                    t = pl.t0 + pl.report.makespan
                    ready.put(pl)
            except BaseException as exc:  # surface planner errors in the caller
                failure.append(exc)
                ready.put(None)
                return
            try:  # plan the next call's first round now (overlaps this call's last round)
                slot = free.get()
                self._prefetch = self.plan(r0 + rounds, t, slot)
            except BaseException as exc:  # e.g. a ConfigError for that round: raised by the next call
                self._prefetch = exc

        th = threading.Thread(target=planner, daemon=True)
        th.start()
        series, pending = [], None
        hs = self.host_s
        for _ in range(rounds):
            t0 = time.perf_counter()
            p = ready.get()
            hs["wait_plan"] = hs.get("wait_plan", 0.0) + time.perf_counter() - t0
            if p is None:
                raise failure[0]
            self.launch(p)
            if pending is not None:   # read the previous round while this one runs
                t0 = time.perf_counter()
                series.extend(self._finish(pending, n_test, on_round, free))
                hs["wait_gpu"] = hs.get("wait_gpu", 0.0) + time.perf_counter() - t0
            pending = p
        series.extend(self._finish(pending, n_test, on_round, free))
        th.join()
        self.round += rounds
        self.now = pending.t0 + pending.report.makespan
        return series

    def _finish(self, p: RoundPlan, n_test: int, on_round, free) -> list:
        self._result_ev[p.slot].synchronize()
        counts = self._correct_pin[p.slot].numpy().copy()
        free.put(p.slot)
        return self._series_entries(p, counts, n_test, on_round)
