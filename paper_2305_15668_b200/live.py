"""Live (real-time) dispatch: the reference's executor manager driven by CUDA
completion events, each client running inside a green-context SM partition
sized by its budget (the paper's runtime, PAPER.md:261,
:337-344; reference live mode comms.py:94-457).

Where the reference's live mode spawns one OS process per executor and
throttles it with an MPS thread percentage, here an executor slot is a
contiguous window of SM groups (`GreenPartitions`), a launch is one
`fedhc_local_train` on that window's stream, "upload" is free (the delta is
already in HBM) and completion is a CUDA event.  The ExecutorManager
(planner.py, reference semantics) decides every launch; the returned
RoundReport is computed from a wall-clock trace with the reference's event
kinds (like `trace_wall.jsonl` of `serve`).

Training results are independent of the dispatch order (every client starts
from the round-start params), so deltas are bit-identical to the batched
path; only timing differs.
"""

from __future__ import annotations

import ctypes as C
import math
import time

import numpy as np
import torch

from . import _abi
from .experiment import CLIENT_DTYPE, DeviceFederation, delta_buffer
from .planner import ClientRequest, ExecutorManager, Participant, RequestKind
from .roundsim import RoundReport, build_round_report
from .spec import ClientProfile, FleetConfig
from .training import check_aggregation, fedavg_device, n_permutations, native_permutations, stable_seed


class GreenPartitions:
    """SM groups of the device and budget -> group-window allocation.

    The native pool (green contexts and their streams, one per group window) is shared per (device, min_sms)
    and lives until process exit: torch keeps events recorded on these streams (pinned-memory copies, the
    caching allocator) past any Python object's lifetime, and destroying a green context under them makes
    later frees fail with "invalid device context".  Each instance keeps its own occupancy counters."""

    _pools: dict = {}

    def __init__(self, device: int = 0, min_sms: int = 8):
        key = (device, min_sms)
        if key not in GreenPartitions._pools:
            pool = C.c_void_p()
            g, spg = C.c_int(), C.c_int()
            _abi.check(_abi.lib.fedhc_gctx_pool_create(device, min_sms, C.byref(pool), C.byref(g), C.byref(spg)))
            GreenPartitions._pools[key] = (pool, g.value, spg.value, {})
        self._pool, self.n_groups, self.sms_per_group, self._streams = GreenPartitions._pools[key]
        self.use = [0] * self.n_groups

    def groups_for(self, budget: float) -> int:
        """Budget b% of the device -> k = max(1, round(b * G / 100)) groups."""
        return max(1, min(self.n_groups, int(round(budget * self.n_groups / 100.0))))

    def stream(self, first: int, count: int) -> int:
        key = (first, count)
        if key not in self._streams:
            s = C.c_void_p()
            _abi.check(_abi.lib.fedhc_gctx_stream(self._pool, first, count, C.byref(s), None))
            self._streams[key] = s.value
        return self._streams[key]

    def stream_rest(self, first: int, count: int) -> tuple[int, int]:
        """(stream, SM count) of a window of `count` groups plus the SMs outside every group."""
        key = (first, -1 - count)
        if key not in self._streams:
            s, n = C.c_void_p(), C.c_int()
            _abi.check(_abi.lib.fedhc_gctx_stream_rest(self._pool, first, count, C.byref(s), C.byref(n)))
            self._streams[key] = (s.value, n.value)
        return self._streams[key]

    def acquire(self, budget: float) -> tuple[int, int, int]:
        """Window with the least overlap with running clients (first fit on ties)."""
        k = self.groups_for(budget)
        best, best_cost = 0, None
        for first in range(self.n_groups - k + 1):
            cost = (max(self.use[first:first + k]), sum(self.use[first:first + k]))
            if best_cost is None or cost < best_cost:
                best, best_cost = first, cost
                if cost == (0, 0):
                    break
        for i in range(best, best + k):
            self.use[i] += 1
        return best, k, self.stream(best, k)

    def release(self, first: int, k: int) -> None:
        for i in range(first, first + k):
            self.use[i] -= 1

    def probe(self, first: int, k: int, blocks: int | None = None) -> set[int]:
        """SM ids a kernel on window [first, first+k) actually ran on (diagnostic)."""
        blocks = blocks or 4 * k * self.sms_per_group
        out = torch.full((blocks,), -1, dtype=torch.int32, device="cuda")
        s = self.stream(first, k)
        _abi.check(_abi.lib.fedhc_probe_smid(s, blocks, out.data_ptr()))
        torch.cuda.ExternalStream(s).synchronize()
        return set(out.cpu().tolist())


class LiveRound:
    """One FL round dispatched in real time onto green-context partitions.

    `engines`: optional per-executor-slot client-model engines (e.g. one `CnnEngine(1, batch, C)` per slot,
    `fed` the matching federation): a launched client then runs that engine's local SGD on its window's stream,
    so a multi-CTA model really runs on (and is sped up or slowed down by) the SM share its budget buys.
    Without engines the client is the reference's logistic model (`fedhc_local_train`, one CTA / cluster).
    """

    def __init__(self, fed: DeviceFederation, fleet: dict[str, ClientProfile], cfg: FleetConfig, lr: float,
                 partitions: GreenPartitions, engines: list | None = None):
        self.fed, self.fleet, self.cfg, self.lr, self.parts = fed, fleet, cfg, float(lr), partitions
        if engines is not None and len(engines) < cfg.max_executors:
            raise ValueError("need one client engine per executor slot")
        self.engines = engines

    def run(self, params: torch.Tensor, participants: list[str], round_index: int = 0, poll_s: float = 2e-5):
        cfg, fed = self.cfg, self.fed
        k = len(participants)
        wls = [self.fleet[c].workload for c in participants]
        seeds = [stable_seed("train", cfg.seed, round_index, c) for c in participants]
        # ---- plan (all permutations at once) + per-client descriptors ----
        meta, rows, perms, rseeds, at = [], [], [], [], 0
        for cid, wl, sd in zip(participants, wls, seeds):
            _, n = fed.offset[cid]
            kp = n_permutations(n, wl.num_samples, wl.batch_size)
            meta.append((at, n, math.ceil(wl.num_samples / wl.batch_size), wl.batch_size))
            rows.append(n)
            perms.append(kp)
            rseeds.append(stable_seed("local_train", sd))
            at += n * kp
        plan = torch.from_numpy(native_permutations(rseeds, rows, perms)).to(fed.x.device) if at else \
            torch.zeros(1, dtype=torch.int32, device=fed.x.device)
        deltas = delta_buffer(max(k, 1), fed.P, fed.x.device)
        desc = fed.descriptor_array(participants, meta, self.lr, deltas, perm_base=plan.data_ptr())
        d_desc = torch.from_numpy(desc.view(np.uint8).copy()).to(fed.x.device)
        torch.cuda.current_stream().synchronize()   # plan, params and descriptors resident before dispatch

        index = {c: i for i, c in enumerate(participants)}
        trace: list[dict] = []
        t_start = time.perf_counter()
        clock = lambda: time.perf_counter() - t_start  # noqa: E731
        mgr = ExecutorManager(cfg.max_executors, cfg.scheduler_kind, cfg.theta, cfg.dynamic_parallelism,
                              trace=lambda e: trace.append({**e, "t": clock()}))
        mgr.begin_round([Participant(c, float(self.fleet[c].resource_budget)) for c in participants])
        running: dict[str, tuple] = {}
        windows: dict[str, tuple[int, int]] = {}
        measured: dict[str, float] = {}

        def launch(entries):
            for entry, _instr in entries:
                cid, budget = entry.client_id, entry.resource_budget
                first, g, s = self.parts.acquire(budget)
                windows[cid] = (first, g)
                ext = torch.cuda.ExternalStream(s)
                ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                ev0.record(ext)
                i = index[cid]
                if self.engines is not None:
                    self.engines[entry.executor_id].local_train(d_desc.data_ptr() + i * CLIENT_DTYPE.itemsize, 1,
                                                                params, meta[i][2], self.lr, use_graph=False,
                                                                stream=s)
                else:
                    fed.launch_train(d_desc.data_ptr() + i * CLIENT_DTYPE.itemsize, 1, params, wls[i].batch_size,
                                     stream=s)
                ev1.record(ext)
                running[cid] = (ev0, ev1, entry.executor_id)
                trace.append({"t": clock(), "kind": "ClientLaunched", "client": cid, "executor": entry.executor_id,
                              "budget": budget, "sm_groups": [first, g]})
                mgr.on_request(ClientRequest(cid, RequestKind.REGISTER), clock())

        launch(mgr.kickoff(0.0))
        while running:
            done = [c for c, (_, ev1, _) in running.items() if ev1.query()]
            if not done:
                time.sleep(poll_s)
                continue
            for cid in sorted(done):
                ev0, ev1, ex = running.pop(cid)
                measured[cid] = ev0.elapsed_time(ev1) / 1e3
                now = clock()
                b = float(self.fleet[cid].resource_budget)
                trace.append({"t": now, "kind": "ClientTrainingComplete", "client": cid, "executor": ex, "budget": b})
                mgr.on_request(ClientRequest(cid, RequestKind.TRAINING_COMPLETE), now)
                trace.append({"t": now, "kind": "ModelUploaded", "client": cid, "executor": ex, "budget": b})
                mgr.on_request(ClientRequest(cid, RequestKind.MODEL_UPLOADED), now)
                self.parts.release(*windows[cid])
                trace.append({"t": now, "kind": "SlotFreed", "client": cid, "executor": ex})
                launch(mgr.on_slot_freed(ex, now))
        if mgr.pending:
            raise RuntimeError(f"round ended with unlaunched participants: {mgr.pending}")
        trace.append({"t": clock(), "kind": "RoundComplete", "round": round_index})
        report: RoundReport = build_round_report(trace, round_index)
        return deltas[:k], report, trace, measured

    def aggregate(self, params: torch.Tensor, deltas: torch.Tensor, participants: list[str]) -> torch.Tensor:
        """Sync FedAvg on the current stream (all client events already completed)."""
        weights = [float(self.fleet[c].workload.num_samples) for c in participants]
        total = check_aggregation(deltas, weights, params.shape)
        coef = torch.tensor([w / total for w in weights], dtype=torch.float64, device=params.device)
        return fedavg_device(deltas, coef, params, params)
