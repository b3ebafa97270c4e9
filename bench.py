#!/usr/bin/env python
"""FedHC round hot-path benchmark on B200 (one JSON line on rank 0).

Workload ("femnist-logreg-c10", BASELINE.json configs[1] with the reference's
model): per GPU 100 participants/round drawn from a 128-per-GPU fleet with
heterogeneous budgets 10..100 (step 10), each a multinomial-logistic client
(F = 784 = 28x28x1, C = 10) with 6400 samples and B = 64, i.e. one local
epoch = 100 SGD steps; theta = 100, resource-aware scheduler, dynamic
parallelism, 18 executors; sync FedAvg + test accuracy every round.

A "step" is one FL round: selection -> native DES schedule -> local SGD of
every participant -> sample-weighted FedAvg -> accuracy.  `value` = client
local-SGD steps per second over the whole job (all ranks), device-resident
(the round plans are uploaded before the timed region).  `e2e` = the same
metric through the public round API with host buffers: selection, DES, PCG64
batch permutations on the host, H2D of the permutations and descriptors,
kernels, D2H of the accuracy count -- every round.

N > 1 (torchrun): every rank trains its own 100 participants (weak scaling);
the only data-path collective is one NCCL all-reduce of the fp64 partial
FedAvg sums per round (+ one int64 all-reduce of the sharded test count).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import random
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

F, C, N_SAMPLES, BATCH, PER_GPU, FLEET_PER_GPU, LR = 784, 10, 6400, 64, 100, 128, 0.1
EXECUTORS, THETA = 18, 100.0
BUDGETS = tuple(range(10, 101, 10))
N_TEST = 16000


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default: 100 rounds for the ~1 ms logistic round, 20 otherwise)")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="bounded CPU-baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sublines", action="store_true", help="skip the c62 / f3072 sub-objects of the round line")
    ap.add_argument("--workload", choices=["round", "cnn", "resnet", "mobilenet", "shufflenet", "fedavg", "gemm", "des",
                                           "live", "data"], default="round",
                    help="round: the FL round (headline); fedavg: config-5 aggregation sweep point")
    ap.add_argument("--fedavg-k", type=int, default=100)
    ap.add_argument("--fedavg-p", type=int, default=11_170_000)
    ap.add_argument("--cnn-samples", type=int, default=6400, help="samples per client for --workload cnn")
    ap.add_argument("--resnet-clients", type=int, default=25, help="ResNet-18 clients per GPU (config 3: 200 / 8)")
    ap.add_argument("--resnet-samples", type=int, default=250, help="samples per ResNet-18 client")
    ap.add_argument("--strong", action="store_true",
                    help="resnet/mobilenet/shufflenet: fixed total participants per round (config 3: --resnet-total "
                         "200 over --gpus N, LPT-sharded) instead of a fixed count per GPU")
    ap.add_argument("--resnet-total", type=int, default=200, help="participants per round with --strong (config 3)")
    ap.add_argument("--mobilenet-clients", type=int, default=100, help="MobileNetV2 participants per GPU per round")
    ap.add_argument("--mobilenet-fleet", type=int, default=1000, help="MobileNetV2 fleet size (config 4: >= 1000)")
    ap.add_argument("--mobilenet-max-samples", type=int, default=1024,
                    help="largest per-client sample count (config 4: uniform choice of 16, 32, ..., 1024)")
    ap.add_argument("--live-samples", type=int, default=640, help="samples per client for --workload live")
    ap.add_argument("--classes", type=int, default=10, help="10 (digits) or 62 (FEMNIST classes, 4-CTA clusters)")
    args = ap.parse_args()
    if args.steps is None:
        args.steps = 100 if (args.workload == "round" and args.impl != "reference") else 20
    return args


def workload_config(n_gpus):
    return {
        "workload": f"femnist-logreg-c{C}: FedHC round of multinomial-logistic clients (reference fl_core model), "
                    f"F=784, C={C}",
        "arithmetic": "fp32 storage/SGD state; products on the bf16 tensor pipe as bf16x3 (hi*hi+hi*mid+mid*hi, "
                      "fp32 accumulate); FedAvg in fp64",
        "participants_per_round": PER_GPU * n_gpus,
        "fleet": FLEET_PER_GPU * n_gpus,
        "samples_per_client": N_SAMPLES,
        "batch": BATCH,
        "local_steps_per_client": math.ceil(N_SAMPLES / BATCH),
        "budgets": "10..100 step 10",
        "theta": THETA,
        "scheduler": "resource-aware, dynamic parallelism",
        "max_executors": EXECUTORS,
        "aggregation": "sync FedAvg (fp64) + accuracy on 16000 test rows every round",
        "parallelism": f"clients sharded over {n_gpus} GPU(s)" + (", NCCL all-reduce of FedAvg partials" if n_gpus > 1
                                                                  else ""),
        "l2": "inputs larger than L2 (2.0 GB of client rows per GPU per round vs 126 MB L2); no flush needed",
    }


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks/throttle sampling DURING the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (FileNotFoundError, OSError):
            self.proc = None
        time.sleep(0.25)
        return self

    def __exit__(self, *exc):
        self.out = ""
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                self.out, _ = self.proc.communicate()

    def summary(self):
        rows = [r.split(",") for r in (self.out or "").strip().splitlines() if r.count(",") >= 8]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].strip().lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# --------------------------------------------------------------------------- CPU reference (oracle port)
_CPU = {}


def _cpu_init():
    # one BLAS thread per worker process (numpy/OpenBLAS is already initialised before the fork)
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)


def _cpu_worker(args):
    from oracle import flmath as fm
    i, seed, params = args
    sh = _CPU["shards"][i % len(_CPU["shards"])]
    return fm.local_sgd(params, sh, N_SAMPLES, BATCH, LR, C, seed=seed)


def cpu_reference(seconds: float, rounds: int | None = None, warmup: int = 0):
    """The reference algorithm (oracle port of fl_core/engine) on the host cores.

    Clients of a round run in a fork pool over all host cores (one BLAS
    thread each); the DES, FedAvg and accuracy run as in the reference.
    Returns (client-steps/s, cores, sample description, rounds timed).
    """
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    import multiprocessing as mp

    from oracle import flmath as fm
    from oracle import orchestration as oc

    cores = len(os.sched_getaffinity(0))
    n_shards = 16
    rng = np.random.default_rng(0)
    means = rng.standard_normal((C, F)) * 3.0
    shards = []
    for _ in range(n_shards):
        y = rng.integers(0, C, N_SAMPLES)
        shards.append(fm.Shard("c", means[y] + rng.standard_normal((N_SAMPLES, F)), y))
    yt = rng.integers(0, C, N_TEST)
    test = fm.Data(means[yt] + rng.standard_normal((N_TEST, F)), yt, C)
    fleet = oc.fleet(FLEET_PER_GPU, 1, budget_levels=BUDGETS, num_samples=N_SAMPLES, batch_size=BATCH)
    by_id = {c.client_id: c for c in fleet}
    ids = sorted(by_id)
    cfg = oc.Config(theta=THETA, max_executors=EXECUTORS, participants_per_round=PER_GPU, seed=1)
    _CPU["shards"] = shards
    _CPU["params"] = fm.zeros_params(F, C)
    pick = random.Random("1:selection")
    steps_per_client = math.ceil(N_SAMPLES / BATCH)
    ctx = mp.get_context("fork")
    done_rounds, t_total = 0, 0.0
    with ctx.Pool(cores, initializer=_cpu_init) as pool:
        r = 0
        while True:
            t0 = time.perf_counter()
            who = pick.sample(ids, PER_GPU)
            oc.simulate_round(by_id, who, cfg)
            base = _CPU["params"]
            deltas = pool.map(_cpu_worker, [(i, fm.seed_of("train", 1, r, c), base) for i, c in enumerate(who)])
            _CPU["params"] = fm.weighted_average(deltas, [float(N_SAMPLES)] * PER_GPU, _CPU["params"])
            fm.accuracy(_CPU["params"], test)
            dt = time.perf_counter() - t0
            r += 1
            if r <= warmup:
                continue
            done_rounds += 1
            t_total += dt
            if (rounds is not None and done_rounds >= rounds) or (rounds is None and t_total >= seconds):
                break
    value = done_rounds * PER_GPU * steps_per_client / t_total
    sample = (f"{done_rounds} full rounds of {PER_GPU} clients x {steps_per_client} steps (F={F}, C={C}, B={BATCH}) "
              f"incl. Python DES, FedAvg and 16000-row accuracy; clients in a fork pool of {cores} processes "
              f"(1 BLAS thread each); shard data cycles over {n_shards} generated shards")
    return value, cores, sample, done_rounds, t_total


# --------------------------------------------------------------------------- GPU arm
def run_ours(args, rank, world, local_rank):
    import torch

    import paper_2305_15668_b200 as fh
    from paper_2305_15668_b200 import _abi
    from paper_2305_15668_b200.experiment import DeviceFederation
    from paper_2305_15668_b200.roundsim import RoundSimulator
    from paper_2305_15668_b200.training import batch_permutations, fedavg_device, stable_seed, stream_ptr

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist_mod
        dist = dist_mod
        dist.init_process_group("nccl", device_id=dev)

    n_fleet = FLEET_PER_GPU * world
    n_part = PER_GPU * world
    P = F * C + C
    steps_per_client = math.ceil(N_SAMPLES / BATCH)

    # ---- device-resident synthetic non-IID data (same seed on every rank) ----
    from paper_2305_15668_b200.devicedata import DeviceFleetData
    from paper_2305_15668_b200.sharding import client_cost, lpt_shards, shard_bounds
    fleet = fh.generate_fleet(fh.DistributionSpec(budget_levels=BUDGETS, num_samples=N_SAMPLES, batch_size=BATCH),
                              n_fleet, 1)
    by_id = {p.client_id: p for p in fleet}
    ids = sorted(by_id)
    data = DeviceFleetData(ids, [by_id[c].workload.num_samples for c in ids], F, C, alpha=0.5, seed=1234,
                           n_test=N_TEST)
    lo, hi = shard_bounds(N_TEST, world, rank)                      # sharded test set
    fed = data.federation(test_slice=(lo, hi))
    cfg = fh.FleetConfig(theta=THETA, max_executors=EXECUTORS, participants_per_round=n_part, seed=1)
    sim = RoundSimulator(by_id)
    stream = torch.cuda.current_stream()

    params = torch.zeros(P, dtype=torch.float64, device=dev)
    partial = torch.empty(P, dtype=torch.float64, device=dev)
    from paper_2305_15668_b200.experiment import delta_buffer
    deltas = delta_buffer(PER_GPU, P, dev)
    weights_coef = torch.full((PER_GPU,), 1.0 / n_part, dtype=torch.float64, device=dev)
    one = torch.ones(1, dtype=torch.float64, device=dev)

    def plan_round(r, selector, now):
        who = selector.sample(ids, n_part)
        rep, _ = sim.run(who, cfg, t0=now, round_index=r, want_trace=False)
        mine = [who[j] for j in lpt_shards([client_cost(by_id[c].workload.num_samples, BATCH) for c in who],
                                           world)[rank]]
        wl = [by_id[c].workload for c in mine]
        seeds = [stable_seed("train", cfg.seed, r, c) for c in mine]
        total = float(sum(float(w.num_samples) for w in (by_id[c].workload for c in who)))
        coef = [float(w.num_samples) / total for w in wl]
        return rep, mine, wl, seeds, coef

    eval_stream = torch.cuda.Stream()
    # the accuracy overlaps the next round's training: with the one-CTA-per-client trainer keep it on the idle
    # SMs; the cluster trainers (62 classes) fill the GPU, so it takes every SM between trainings (as
    # FederatedRunner._side_ctas)
    from paper_2305_15668_b200.training import train_sms_per_client
    n_sms = torch.cuda.get_device_properties(dev).multi_processor_count
    eval_ctas = n_sms if train_sms_per_client(F, C) > 1 else max(8, n_sms - PER_GPU)
    eval_done = [None]

    def device_round(mine_desc, coef_dev, correct):
        """train -> FedAvg partial -> (all-reduce) -> apply -> sharded accuracy; returns train events.
        Single GPU: the accuracy runs on its own stream, overlapping the next round's training (both only
        read the params; the next FedAvg waits for it), as FederatedRunner does."""
        main = torch.cuda.current_stream()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        fed.launch_train(mine_desc.data_ptr(), PER_GPU, params, BATCH)
        ev1.record()
        if world == 1:
            if eval_done[0] is not None:
                main.wait_event(eval_done[0])
            fedavg_device(deltas, coef_dev, params, params)
            agg = torch.cuda.Event()
            agg.record(main)
            eval_stream.wait_event(agg)
            _abi.check(_abi.lib.fedhc_eval_ctas(fed.x_test.data_ptr(), fed.y_test.data_ptr(), fed.n_test, F, C,
                                                params.data_ptr(), correct.data_ptr(), eval_ctas,
                                                eval_stream.cuda_stream))
            done = torch.cuda.Event()
            done.record(eval_stream)
            eval_done[0] = done
            return ev0, ev1
        fedavg_device(deltas, coef_dev, None, partial)
        dist.all_reduce(partial)
        fedavg_device(partial.view(1, -1), one, params, params)
        _abi.check(_abi.lib.fedhc_eval(fed.x_test.data_ptr(), fed.y_test.data_ptr(), fed.n_test, F, C,
                                       params.data_ptr(), correct.data_ptr(), stream_ptr()))
        dist.all_reduce(correct)
        return ev0, ev1

    def join_eval():
        if eval_done[0] is not None:
            torch.cuda.current_stream().wait_event(eval_done[0])

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # ---------------- value: device-resident rounds ----------------
    total_rounds = args.warmup + args.steps
    selector = random.Random(f"{cfg.seed}:selection")
    plans, now = [], 0.0
    for r in range(total_rounds):
        rep, mine, wl, seeds, coef = plan_round(r, selector, now)
        now += rep.makespan
        packed, meta = fed.plan(mine, wl, seeds)
        perm_dev = torch.from_numpy(packed).to(dev)
        fed._perm_dev = perm_dev
        desc = fed.descriptors(mine, meta, LR, deltas)
        plans.append((perm_dev, desc, torch.tensor(coef, dtype=torch.float64, device=dev)))
    counts = torch.zeros(total_rounds, dtype=torch.int64, device=dev)
    for r in range(args.warmup):
        device_round(plans[r][1], plans[r][2], counts[r:r + 1])
    barrier()
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    train_events = []
    with ClockSampler(local_rank) as clocks:
        barrier()
        t_start.record()
        for r in range(args.warmup, total_rounds):
            train_events.append(device_round(plans[r][1], plans[r][2], counts[r:r + 1]))
        join_eval()  # the last round's accuracy belongs to the timed region
        t_end.record()
        barrier()
    ms = t_start.elapsed_time(t_end)
    train_ms = float(np.mean([a.elapsed_time(b) for a, b in train_events]))
    if dist is not None:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    accuracy_last = counts[-1].item() / N_TEST
    launches_per_round = 3 + (1 if world > 1 else 0)  # train, FedAvg (+apply), eval
    total_steps = args.steps * n_part * steps_per_client
    value = total_steps / (ms / 1e3)

    # ---------------- e2e: public round API with host buffers ----------------
    # FederatedRunner: per round the host plans (selection, native DES, seeds, PCG64 permutations into
    # pinned memory), copies the plan H2D, launches train/FedAvg/(all-reduce)/eval and reads the
    # accuracy count back (D2H); planning of round r+1 overlaps the GPU work of round r.
    from paper_2305_15668_b200.experiment import FederatedRunner
    runner = FederatedRunner(fed, by_id, cfg, LR, world=world, rank=rank, group=None, test_sharded=True)
    runner.run(args.warmup, n_test_total=N_TEST)
    barrier()
    trace = os.environ.get("FEDHC_TRACE")  # optional: kernel timeline of the e2e rounds (torch.profiler / CUPTI)
    if trace:
        prof = torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA,
                                                  torch.profiler.ProfilerActivity.CPU])
        prof.__enter__()
    e0 = time.perf_counter()
    series = runner.run(args.steps, n_test_total=N_TEST)
    barrier()
    e2e_s = time.perf_counter() - e0
    if trace:
        prof.__exit__(None, None, None)
        prof.export_chrome_trace(trace)
    h2d, d2h = runner.h2d_bytes, runner.d2h_bytes
    host_ms = {k: round(v / (args.steps + args.warmup) * 1e3, 4) for k, v in runner.host_s.items()}
    if dist is not None:
        t = torch.tensor([e2e_s], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = total_steps / e2e_s

    # ---------------- roofline of the dominant kernel (train) ----------------
    from benchlib import roofline_entry
    bytes_per_launch = PER_GPU * steps_per_client * BATCH * (4 * F + 8) + PER_GPU * P * 12
    roof = roofline_entry(bytes_per_launch, train_ms, ROOT,
                          kernel=("train_pipe2_kernel" if fed.x_split is not None else "train_pipe_kernel") if C <= 16
                          else "train_fused_kernel")

    result = {
        "metric": "client local-steps/sec (FedHC round: local SGD of all participants + FedAvg + accuracy)",
        "value": value,
        "unit": "client-steps/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16x3",  # bf16 hi/mid products (hi*hi + hi*mid + mid*hi), fp32 accumulate and SGD state
        "data": "synthetic, generated in HBM: Gaussian class clusters + Dirichlet(0.5) non-IID client label mix "
                "(reference distributions, not the reference's RNG stream)",
        "config": workload_config(world),
        "rounds_per_sec": args.steps / (ms / 1e3),
        "train_kernel_ms": train_ms,
        "accuracy_last_round": accuracy_last,
        "e2e": {"value": e2e_value, "unit": "client-steps/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "rounds_per_sec": args.steps / e2e_s,
                "api": "paper_2305_15668_b200.experiment.FederatedRunner.run (pipelined host planning)",
                "host_ms_per_round": host_ms,
                "accuracy_last_round": series[-1][1] if series else None},
        "roofline": roof,
        "clocks": clocks.summary(),
        "gpu_launches": launches_per_round * args.steps,
    }
    if C == 10 and not args.no_sublines:
        # the other reference-model shapes the round is quoted on: FEMNIST's 62 classes (train_c64_kernel,
        # 2-CTA tcgen05 clusters), the CIFAR-shaped F = 3072 model (train_tc_kernel, 8-CTA clusters), and
        # config 2's FEMNIST CNN
        result["c62"] = kernel_subline(62, 784, PER_GPU, N_SAMPLES, 5, 2)
        result["f3072"] = kernel_subline(10, 3072, PER_GPU, 640, 5, 2)
        result["cnn"] = cnn_subline(62, PER_GPU, 640, 3, 1)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, cores, sample, _, _ = cpu_reference(args.cpu_seconds, warmup=1)
        result["cpu_baseline"] = {"value": v, "unit": "client-steps/s", "cores": cores, "kind": "port",
                                  "sample": sample}
    if dist is not None:
        dist.destroy_process_group()
    return result


def kernel_subline(C_, F_, n_clients, n_samp, rounds, warm, fleet_seed=1):
    """Device-resident local-SGD rounds at another reference-model shape (same round structure, same
    100-participant selection stream), for the driver-visible sub-objects of the default bench line:
    "c62" (FEMNIST's 62 classes) and "f3072" (the CIFAR-shaped reference model).
    Times fedhc_local_train with CUDA events on its stream; HBM roofline by the same algorithmic bytes."""
    import torch
    import paper_2305_15668_b200 as fh
    from paper_2305_15668_b200 import _abi
    from paper_2305_15668_b200.devicedata import DeviceFleetData
    from paper_2305_15668_b200.experiment import delta_buffer
    from paper_2305_15668_b200.training import fedavg_device, stable_seed, stream_ptr
    from benchlib import roofline_entry

    dev = torch.device("cuda", torch.cuda.current_device())
    fleet = fh.generate_fleet(fh.DistributionSpec(budget_levels=BUDGETS, num_samples=n_samp, batch_size=BATCH),
                              FLEET_PER_GPU, fleet_seed)
    by_id = {p.client_id: p for p in fleet}
    ids = sorted(by_id)
    data = DeviceFleetData(ids, [by_id[c].workload.num_samples for c in ids], F_, C_, alpha=0.5, seed=1234,
                           n_test=4096)
    fed = data.federation()
    P = F_ * C_ + C_
    params = torch.zeros(P, dtype=torch.float64, device=dev)
    deltas = delta_buffer(n_clients, P, dev)
    selector = random.Random(f"{fleet_seed}:selection")
    plans = []
    for r in range(rounds + warm):
        mine = selector.sample(ids, n_clients)
        wl = [by_id[c].workload for c in mine]
        packed, meta = fed.plan(mine, wl, [stable_seed("train", fleet_seed, r, c) for c in mine])
        perm_dev = torch.from_numpy(packed).to(dev)
        fed._perm_dev = perm_dev
        plans.append((perm_dev, fed.descriptors(mine, meta, LR, deltas)))
    coef = torch.full((n_clients,), 1.0 / n_clients, dtype=torch.float64, device=dev)
    evs = []
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for i, (_, desc) in enumerate(plans):
        if i == warm:
            torch.cuda.synchronize()
            t0.record()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fed.launch_train(desc.data_ptr(), n_clients, params, BATCH)
        b.record()
        if i >= warm:
            evs.append((a, b))
        fedavg_device(deltas, coef, params, params)
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / rounds
    train_ms = float(np.mean([a.elapsed_time(b) for a, b in evs]))
    steps = n_clients * math.ceil(n_samp / BATCH)
    bytes_launch = n_clients * math.ceil(n_samp / BATCH) * BATCH * (4 * F_ + 8) + n_clients * P * 12
    kern = ("train_c64_kernel" if F_ <= 784 else "train_tc_kernel") if (F_ > 784 or C_ > 32) else "train_pipe_kernel"
    return {"workload": f"femnist-logreg F={F_}, C={C_}: {n_clients} clients x {n_samp} samples, B={BATCH}, "
                        f"local SGD + FedAvg (device-resident rounds)",
            "value": steps / (ms / 1e3), "unit": "client-steps/s", "ms_per_round": ms, "train_kernel_ms": train_ms,
            "rounds": rounds, "roofline": roofline_entry(bytes_launch, train_ms, ROOT, kernel=kern)}


def cnn_subline(nc, n_clients, n_samp, rounds, warm, fleet_seed=1):
    """BASELINE config 2's model (FEMNIST CNN, tcgen05 grouped implicit GEMMs, one CUDA graph per round) as a
    driver-visible sub-object of the default line: device-resident rounds of n_clients x n_samp samples (the
    full config-2 shape is `--workload cnn`), local SGD + FedAvg + accuracy, train phase timed with CUDA events;
    tensor roofline by the algorithmic FLOPs, HBM roofline by the fp32 master traffic."""
    import torch
    import paper_2305_15668_b200 as fh
    from paper_2305_15668_b200.cnn import CnnFederation, init_cnn_params
    from paper_2305_15668_b200.devicedata import DeviceFleetData
    from paper_2305_15668_b200.experiment import delta_buffer
    from paper_2305_15668_b200.training import fedavg_device, stable_seed
    from benchlib import hbm_peak

    dev = torch.device("cuda", torch.cuda.current_device())
    bs, lr = 64, 0.01
    fleet = fh.generate_fleet(fh.DistributionSpec(budget_levels=BUDGETS, num_samples=n_samp, batch_size=bs),
                              FLEET_PER_GPU, fleet_seed)
    by_id = {p.client_id: p for p in fleet}
    ids = sorted(by_id)
    data = DeviceFleetData(ids, [by_id[c].workload.num_samples for c in ids], 784, nc, alpha=0.5, seed=1234,
                           n_test=4096)
    fed = CnnFederation.from_arrays(data.x, data.y, data.offsets, data.x_test, data.y_test, nc).attach_engine(
        n_clients, bs)
    params = torch.tensor(fed.layout.to_padded(init_cnn_params(nc, 1)), dtype=torch.float64, device=dev)
    deltas = delta_buffer(n_clients, fed.P, dev)
    selector = random.Random(f"{fleet_seed}:selection")
    plans = []
    for r in range(rounds + warm):
        mine = selector.sample(ids, n_clients)
        wl = [by_id[c].workload for c in mine]
        packed, meta = fed.plan(mine, wl, [stable_seed("train", fleet_seed, r, c) for c in mine])
        perm_dev = torch.from_numpy(packed).to(dev)
        fed._perm_dev = perm_dev
        plans.append((perm_dev, fed.descriptors(mine, meta, lr, deltas), max(m[2] for m in meta)))
    coef = torch.full((n_clients,), 1.0 / n_clients, dtype=torch.float64, device=dev)
    counts = torch.zeros(rounds + warm, dtype=torch.int64, device=dev)
    evs = []
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for i, (_, desc, steps) in enumerate(plans):
        if i == warm:
            torch.cuda.synchronize()
            t0.record()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fed.engine.local_train(desc.data_ptr(), n_clients, params, steps, lr, True)
        b.record()
        if i >= warm:
            evs.append((a, b))
        fedavg_device(deltas, coef, params, params)
        fed.engine.correct_into(params, fed.x_test, fed.y_test, counts[i:i + 1])
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / rounds
    train_ms = float(np.mean([a.elapsed_time(b) for a, b in evs]))
    steps = n_clients * math.ceil(n_samp / bs)
    flops = cnn_flop_per_sample(nc) * n_clients * n_samp
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        peak, src = float(peaks["bf16_tflops"]), "MEASURED_PEAKS.json bf16_tflops (cuBLAS, measured)"
    except (OSError, KeyError, ValueError):
        peak, src = 1590.0, "fallback 1.59 PFLOP/s (B200_PROFILING.md)"
    tf = flops / (train_ms * 1e-3) / 1e12
    hbm_v, hbm_src = hbm_peak(ROOT)
    hbm_alg = float(steps * (8 * fed.layout.canonical_count + bs * (784 * 4 + 4)))
    return {"workload": f"femnist-cnn-c{nc} (BASELINE config 2's model): {n_clients} clients x {n_samp} samples, "
                        f"B={bs}, local SGD + FedAvg + accuracy (device-resident rounds; the full config-2 round is "
                        f"--workload cnn)",
            "value": steps / (ms / 1e3), "unit": "client-steps/s", "ms_per_round": ms, "train_ms": train_ms,
            "rounds": rounds, "dtype": "bf16 operands (tcgen05), fp32 accumulation and masters",
            "roofline_tensor": {"bound": "tensor", "achieved": tf, "peak": peak, "unit": "TFLOP/s",
                                "frac": tf / peak, "algorithmic_flop_per_launch": flops, "peak_source": src,
                                "kernel": "train phase (one CUDA graph of grouped_gemm_kernel + conv1/pool/CE)"},
            "roofline": {"bound": "hbm", "achieved": hbm_alg / (train_ms * 1e-3) / 1e9, "peak": hbm_v,
                         "unit": "GB/s", "frac": hbm_alg / (train_ms * 1e-3) / 1e9 / hbm_v,
                         "algorithmic_bytes_per_launch": hbm_alg, "peak_source": hbm_src},
            "accuracy_last_round": counts[-1].item() / 4096}


def run_live(args, rank, world, local_rank):
    """--workload live: the paper's runtime -- every launch decided in real time by the
    executor manager (executor_manager.py:81-238) on CUDA completion events, each client's FEMNIST CNN (config 2's
    model) running on the green-context SM window its budget buys (k = round(b * G / 100) groups of 8 SMs).
    value = client local-SGD steps per second of wall time (host-driven dispatch, so wall-clock, not events);
    also reported: how the measured per-client GPU times track the DES's simulated per-client times (Pearson r of
    measured vs simulated, and of measured vs 1 / budget), and the live vs simulated makespan."""
    import torch
    import paper_2305_15668_b200 as fh
    from paper_2305_15668_b200.cnn import CnnEngine, CnnFederation, init_cnn_params
    from paper_2305_15668_b200.devicedata import DeviceFleetData
    from paper_2305_15668_b200.live import GreenPartitions, LiveRound
    from paper_2305_15668_b200.roundsim import RoundSimulator

    if world > 1:
        raise SystemExit("--workload live runs on one GPU (a round's partitions are one device's SMs)")
    torch.cuda.set_device(local_rank)
    nc, n_samp, bs, lr = 62, args.live_samples, 64, 0.01
    fleet = fh.generate_fleet(fh.DistributionSpec(budget_levels=BUDGETS, num_samples=n_samp, batch_size=bs),
                              FLEET_PER_GPU, 1)
    by_id = {p.client_id: p for p in fleet}
    ids = sorted(by_id)
    data = DeviceFleetData(ids, [by_id[c].workload.num_samples for c in ids], 784, nc, alpha=0.5, seed=1234,
                           n_test=1024)
    fed = CnnFederation.from_arrays(data.x, data.y, data.offsets, data.x_test, data.y_test, nc).attach_engine(1, bs)
    cfg = fh.FleetConfig(theta=THETA, max_executors=EXECUTORS, participants_per_round=PER_GPU, seed=1)
    parts = GreenPartitions(local_rank, 8)
    engines = [CnnEngine(1, bs, nc) for _ in range(cfg.max_executors)]
    live = LiveRound(fed, by_id, cfg, lr, parts, engines=engines)
    sim = RoundSimulator(by_id)
    params = torch.tensor(fed.layout.to_padded(init_cnn_params(nc, 1)), dtype=torch.float64, device="cuda")
    selector = random.Random(f"{cfg.seed}:selection")
    steps_per_client = math.ceil(n_samp / bs)
    meas, simt, budg, spans = [], [], [], []
    wall = 0.0
    for r in range(args.warmup + args.steps):
        who = selector.sample(ids, PER_GPU)
        t0 = time.perf_counter()
        deltas, rep, trace, measured = live.run(params, who, round_index=r)
        live.aggregate(params, deltas, who)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if r < args.warmup:
            continue
        wall += dt
        srep, _ = sim.run(who, cfg, t0=0.0, round_index=r, want_trace=False)
        spans.append((rep.makespan, srep.makespan))
        for c in who:
            meas.append(measured[c])
            simt.append(srep.per_client_end[c] - srep.per_client_start[c])
            budg.append(float(by_id[c].resource_budget))
    meas, simt, budg = np.array(meas), np.array(simt), np.array(budg)
    r_sim = float(np.corrcoef(meas, simt)[0, 1])
    r_inv = float(np.corrcoef(meas, 1.0 / budg)[0, 1])
    by_b = {int(b): float(np.median(meas[budg == b]) * 1e3) for b in sorted(set(budg.tolist()))}
    total_steps = args.steps * PER_GPU * steps_per_client
    value = total_steps / wall
    return {
        "metric": "client local-steps/sec (FedHC round: local SGD of all participants + FedAvg + accuracy)",
        "value": value, "unit": "client-steps/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": wall / args.steps * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic FEMNIST-shaped rows generated in HBM; random-init FEMNIST CNN",
        "config": {"workload": f"live-femnist-cnn-c{nc}: live dispatch (executor manager on CUDA completion "
                               f"events), clients on green-context SM windows sized by budget",
                   "participants_per_round": PER_GPU, "fleet": FLEET_PER_GPU, "samples_per_client": n_samp,
                   "batch": bs, "budgets": "10..100 step 10", "theta": THETA, "max_executors": EXECUTORS,
                   "sm_groups": parts.n_groups, "sms_per_group": parts.sms_per_group,
                   "timing": "wall clock per round (host-driven dispatch, round = live.run + FedAvg)"},
        "budget_physics": {"pearson_measured_vs_des_client_time": r_sim,
                           "pearson_measured_vs_inverse_budget": r_inv,
                           "median_client_ms_by_budget": by_b,
                           "makespan_live_s_vs_des_s": [float(np.mean([a for a, _ in spans])),
                                                        float(np.mean([b for _, b in spans]))]},
        "gpu_launches": args.steps * (PER_GPU * engines[0].launches_per_round(steps_per_client) + 1),
    }


def run_fedavg(args, rank, world, local_rank):
    """Config 5: K fp32 client deltas of P params -> fp64 FedAvg (one point of the sweep).

    Each rank aggregates its K deltas (weak scaling) and the ranks all-reduce
    the fp64 partial sums over NCCL.  Inputs (K*P*4 bytes) exceed L2.
    """
    import torch

    from paper_2305_15668_b200.training import fedavg_device

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist_mod
        dist = dist_mod
        dist.init_process_group("nccl", device_id=dev)
    K, P = args.fedavg_k, args.fedavg_p
    g = torch.Generator(device=dev).manual_seed(rank)
    deltas = torch.empty(K, (P + 3) // 4 * 4, device=dev)[:, :P]
    for k in range(K):
        deltas[k].normal_(0.0, 1e-3, generator=g)
    base = torch.randn(P, device=dev, dtype=torch.float64, generator=g)
    w = torch.randint(1, 1025, (K * world,), generator=torch.Generator().manual_seed(0)).double()
    coef = (w / w.sum())[rank * K:(rank + 1) * K].to(dev)
    out = torch.empty_like(base)
    partial = torch.empty_like(base)
    one = torch.ones(1, dtype=torch.float64, device=dev)

    def step():
        if world == 1:
            fedavg_device(deltas, coef, base, out)
        else:
            fedavg_device(deltas, coef, None, partial)
            dist.all_reduce(partial)
            fedavg_device(partial.view(1, -1), one, base, out)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clocks:
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    if dist:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.destroy_process_group()
    from benchlib import roofline_entry
    alg_bytes = K * P * 4 + 2 * P * 8
    res = {
        "metric": "FedAvg aggregated client-delta bytes/sec (config 5)",
        "value": world * alg_bytes / (ms * 1e-3) / 1e9, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic N(0,1e-3) fp32 deltas, N(0,1) fp64 base",
        "config": {"workload": f"fedavg K={K} P={P} per GPU", "l2": "inputs larger than L2"},
        "roofline": roofline_entry(alg_bytes, ms, ROOT, kernel="fedavg_kernel"),
        "clocks": clocks.summary(), "gpu_launches": args.steps * (1 if world == 1 else 2),
    }
    return res


def run_data(args, local_rank):
    """SURVEY §8f rank 2 (fl_core.py:41-115): the reference experiment's synthetic dataset + non-IID partition at
    fleet scale, bit-identical to the reference, built in HBM (devicedata.reference_federation: host centres /
    labels / partition bookkeeping, device ziggurat normals).  value = dataset rows produced per second; the
    CPU baseline runs the reference algorithm (numpy make_synthetic_dataset + partition_noniid, the oracle's
    restatement) on a bounded sample."""
    import torch

    from paper_2305_15668_b200.devicedata import reference_federation
    torch.cuda.set_device(local_rank)
    n_clients, n_samp, F, C = 1000, 600, 784, 10
    clients = [(f"c{i:04d}", n_samp) for i in range(n_clients)]
    n_total = math.ceil(n_clients * n_samp / 0.8)

    def build(seed):
        fed = reference_federation(clients, F, C, n_total, seed, 0.5, seed + 1)
        torch.cuda.synchronize()
        return fed

    for i in range(args.warmup):
        build(100 + i)
    times = []
    with ClockSampler(local_rank) as clocks:
        for i in range(args.steps):
            t = time.perf_counter()
            build(1000 + i)
            times.append(time.perf_counter() - t)
    s_med = float(np.median(times))
    res = {
        "metric": "synthetic dataset + non-IID partition rows generated per second (fl_core.py:41-115)",
        "value": n_total / s_med, "unit": "rows/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": s_med * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "the reference's own synthetic data, bit for bit (numpy PCG64 streams reproduced)",
        "config": {"workload": f"reference experiment data: {n_clients} clients x {n_samp} samples, F={F}, C={C}, "
                               f"n_total={n_total} (test = n_total // 5), Dirichlet(0.5)",
                   "timing": "wall clock per build incl. host labels / partition and H2D (device-synchronised)"},
        "clocks": clocks.summary(),
        # per build: fedhc_pcg64_standard_normal's two kernels per 2^18-row chunk, fedhc_x_split once
        "gpu_launches": args.steps * (2 * math.ceil(n_total / (1 << 18)) + 1),
    }
    if not args.no_cpu_baseline:
        import oracle.flmath as fm
        n_small = max(10, int(n_total * 0.05))
        small = [(c, n) for c, n in clients[:int(n_clients * 0.05)]]
        t = time.perf_counter()
        trn, _ = fm.synthetic(F, C, n_small, 7)
        fm.dirichlet_partition(trn, small, 0.5, 8)
        dt = time.perf_counter() - t
        res["cpu_baseline"] = {"value": n_small / dt, "unit": "rows/s", "cores": 1, "kind": "port",
                               "sample": f"{n_small} rows ({len(small)} clients) through the oracle's numpy "
                                         f"restatement of make_synthetic_dataset + partition_noniid"}
    return res


def run_gemm(args, rank, world, local_rank):
    """tcgen05 grouped GEMM primitive: per-client FC1 of the FEMNIST CNN head (3136 -> 2048) on a
    256-sample slab, all clients of a round in one launch.  Reported against the measured bf16 peak."""
    import torch

    from paper_2305_15668_b200 import _abi
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    G, M, N, K = 100, 2048, 256, 3136
    g = torch.Generator(device=dev).manual_seed(0)
    A = torch.randn(G, M, K, device=dev, generator=g).to(torch.bfloat16)
    B = torch.randn(G, N, K, device=dev, generator=g).to(torch.bfloat16)
    D = torch.empty(G, M, N, device=dev)
    sp = torch.cuda.current_stream().cuda_stream

    def step():
        _abi.check(_abi.lib.fedhc_gemm_bf16_tn(G, M, N, K, A.data_ptr(), B.data_ptr(), D.data_ptr(), sp))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clocks:
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    flops = 2.0 * G * M * N * K
    tf = flops / (ms * 1e-3) / 1e12
    import json as _json
    try:
        peaks = _json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        peak, src = float(peaks["bf16_tflops"]), "MEASURED_PEAKS.json bf16_tflops (cuBLAS burst)"
    except (OSError, KeyError, ValueError):
        peak, src = 1590.0, "fallback 1.59 PFLOP/s (B200_PROFILING.md)"
    return {
        "metric": "grouped GEMM TFLOP/s (tcgen05, per-client FC layer)", "value": tf, "unit": "TFLOP/s",
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": f"grouped GEMM G={G} M={M} N={N} K={K} (D = A.B^T per group)"},
        "roofline": {"bound": "tensor", "achieved": tf, "peak": peak, "unit": "TFLOP/s", "frac": tf / peak,
                     "traffic": None, "kernel": "grouped_gemm_kernel", "peak_source": src},
        "clocks": clocks.summary(), "gpu_launches": args.steps,
    }


def run_des(args):
    """Round control plane (engine.run_round: schedulers + executor manager + DES + metrics) at
    N = 100 / 1000 / 2000 participants (resource-aware, theta = 100, 16 executors): native
    C++ DES vs the reference algorithm (oracle port, Python), same inputs, bit-identical reports."""
    import paper_2305_15668_b200 as fh
    from oracle import orchestration as oc
    from paper_2305_15668_b200.roundsim import RoundSimulator
    rows = []
    for n in (100, 1000, 2000):
        dist = dict(budget_levels=(10, 15, 30, 40, 50, 65, 80))
        pf = fh.generate_fleet(fh.DistributionSpec(**dist), n, 17)
        of = oc.fleet(n, 17, **dist)
        ids = sorted(p.client_id for p in pf)
        cfg = dict(theta=100.0, max_executors=16, seed=17)
        sim = RoundSimulator({p.client_id: p for p in pf})
        reps = max(3, args.steps)
        t0 = time.perf_counter()
        for _ in range(reps):
            rep, _ = sim.run(ids, fh.FleetConfig(**cfg), want_trace=False)
        native = (time.perf_counter() - t0) / reps
        t0 = time.perf_counter()
        orep, _ = oc.simulate_round({c.client_id: c for c in of}, ids, oc.Config(**cfg))
        ref = time.perf_counter() - t0
        assert rep.makespan == orep["makespan"] and rep.vacancy_area == orep["vacancy_area"]
        rows.append({"participants": n, "native_ms": native * 1e3, "reference_ms": ref * 1e3,
                     "speedup": ref / native, "makespan_s": rep.makespan})
    top = rows[-1]
    return {
        "metric": "round control-plane rounds/sec (schedule + executor manager + DES + metrics)",
        "value": 1e3 / top["native_ms"], "unit": "rounds/s", "n_gpus": 0, "steps": args.steps, "warmup": 0,
        "ms_per_step": top["native_ms"], "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic fleet (generate_fleet, seed 17)",
        "config": {"workload": "engine.run_round at N=2000 participants, resource-aware, theta=100, 16 executors",
                   "sweep": rows},
        "cpu_baseline": {"value": 1e3 / top["reference_ms"], "unit": "rounds/s", "cores": 1, "kind": "port",
                         "sample": "one round per N with the oracle's Python DES (reference algorithm)"},
    }


CNN_FLOP_PER_SAMPLE = 102.0e6   # FEMNIST CNN fwd+bwd (no conv1 dgrad), C=62 (torch FlopCounter)


def cnn_flop_per_sample(n_classes: int) -> float:
    """Algorithmic (unpadded) fwd + wgrad + dgrad FLOPs of one FEMNIST-CNN sample."""
    fwd = [2 * 784 * 32 * 25, 2 * 196 * 64 * 800, 2 * 3136 * 2048, 2 * 2048 * n_classes]
    return float(sum(fwd) * 2 + sum(fwd[1:]))     # forward + weight grads + input grads of layers 2..4


def cnn_cpu_reference(seconds: float, n_classes: int, batch: int):
    """FEMNIST-CNN local SGD on the host cores (torch CPU, all threads): the CPU restatement (no reference CNN)."""
    import torch
    import torch.nn as nn
    cores = len(os.sched_getaffinity(0))
    torch.set_num_threads(cores)
    torch.manual_seed(0)
    model = nn.Sequential(nn.Conv2d(1, 32, 5, padding=2), nn.ReLU(), nn.MaxPool2d(2),
                          nn.Conv2d(32, 64, 5, padding=2), nn.ReLU(), nn.MaxPool2d(2), nn.Flatten(),
                          nn.Linear(3136, 2048), nn.ReLU(), nn.Linear(2048, n_classes))
    opt = torch.optim.SGD(model.parameters(), lr=0.01)
    x = torch.randn(1024, 1, 28, 28)
    y = torch.randint(0, n_classes, (1024,))
    lossf = nn.CrossEntropyLoss()

    def one(i):
        s = (i * batch) % (1024 - batch)
        opt.zero_grad(set_to_none=True)
        lossf(model(x[s:s + batch]), y[s:s + batch]).backward()
        opt.step()

    for i in range(3):
        one(i)
    n, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < seconds:
        one(n)
        n += 1
    dt = time.perf_counter() - t0
    return n / dt, cores, (f"{n} local SGD steps (B={batch}) of one FEMNIST-CNN client, torch CPU fp32 with "
                           f"{cores} threads (CPU restatement: the reference has no CNN)"), n, dt


def run_cnn(args, rank, world, local_rank):
    """BASELINE config 2 with its named model: FEMNIST CNN clients, 100 participants/round per GPU,
    heterogeneous budgets 10..100, the round DES, batched local SGD on the tcgen05 engine, FedAvg, accuracy."""
    import torch

    import paper_2305_15668_b200 as fh
    from paper_2305_15668_b200.cnn import CnnFederation, init_cnn_params
    from paper_2305_15668_b200.devicedata import DeviceFleetData
    from paper_2305_15668_b200.experiment import delta_buffer
    from paper_2305_15668_b200.roundsim import RoundSimulator
    from paper_2305_15668_b200.sharding import client_cost, lpt_shards, shard_bounds
    from paper_2305_15668_b200.training import fedavg_device, stable_seed

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist_mod
        dist = dist_mod
        dist.init_process_group("nccl", device_id=dev)
    nc, n_samp, bs, per_gpu, lr = args.classes, args.cnn_samples, 64, PER_GPU, 0.01
    n_part, n_fleet = per_gpu * world, FLEET_PER_GPU * world
    steps_per_client = math.ceil(n_samp / bs)
    fleet = fh.generate_fleet(fh.DistributionSpec(budget_levels=BUDGETS, num_samples=n_samp, batch_size=bs),
                              n_fleet, 1)
    by_id = {p.client_id: p for p in fleet}
    ids = sorted(by_id)
    n_test = 4096
    data = DeviceFleetData(ids, [by_id[c].workload.num_samples for c in ids], 784, nc, alpha=0.5, seed=1234,
                           n_test=n_test)
    lo, hi = shard_bounds(n_test, world, rank)
    fed = CnnFederation.from_arrays(data.x, data.y, data.offsets, data.x_test[lo:hi].contiguous(),
                                    data.y_test[lo:hi].contiguous(), nc).attach_engine(per_gpu, bs)
    P = fed.P
    params = torch.tensor(fed.layout.to_padded(init_cnn_params(nc, 1)), dtype=torch.float64, device=dev)
    deltas = delta_buffer(per_gpu, P, dev)
    partial = torch.empty(P, dtype=torch.float64, device=dev)
    one = torch.ones(1, dtype=torch.float64, device=dev)
    cfg = fh.FleetConfig(theta=THETA, max_executors=EXECUTORS, participants_per_round=n_part, seed=1)
    sim = RoundSimulator(by_id)
    selector = random.Random(f"{cfg.seed}:selection")
    total_rounds = args.warmup + args.steps

    def plan_round(r, now):
        who = selector.sample(ids, n_part)
        rep, _ = sim.run(who, cfg, t0=now, round_index=r, want_trace=False)
        mine = [who[j] for j in lpt_shards([client_cost(by_id[c].workload.num_samples, bs) for c in who],
                                           world)[rank]]
        wl = [by_id[c].workload for c in mine]
        seeds = [stable_seed("train", cfg.seed, r, c) for c in mine]
        total = float(sum(float(by_id[c].workload.num_samples) for c in who))
        coef = torch.tensor([float(w.num_samples) / total for w in wl], dtype=torch.float64, device=dev)
        return rep, mine, wl, seeds, coef

    def coef_of(mine):
        total = float(n_part * n_samp)
        return torch.tensor([float(by_id[c].workload.num_samples) / total for c in mine], dtype=torch.float64,
                            device=dev)

    def aggregate(coef):
        if world == 1:
            fedavg_device(deltas, coef, params, params)
        else:
            fedavg_device(deltas, coef, None, partial)
            dist.all_reduce(partial)
            fedavg_device(partial.view(1, -1), one, params, params)

    # ---- value: device-resident rounds (plans uploaded before timing) ----
    plans, now = [], 0.0
    for r in range(total_rounds):
        rep, mine, wl, seeds, coef = plan_round(r, now)
        now += rep.makespan
        packed, meta = fed.plan(mine, wl, seeds)
        perm_dev = torch.from_numpy(packed).to(dev)
        fed._perm_dev = perm_dev
        desc = fed.descriptors(mine, meta, lr, deltas)
        plans.append((perm_dev, desc, coef, max(m[2] for m in meta)))
    counts = torch.zeros(total_rounds, dtype=torch.int64, device=dev)

    def device_round(r):
        _, desc, coef, steps = plans[r]
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        fed.engine.local_train(desc.data_ptr(), per_gpu, params, steps, lr, True)
        ev1.record()
        aggregate(coef)
        fed.engine.correct_into(params, fed.x_test, fed.y_test, counts[r:r + 1])
        if world > 1:
            dist.all_reduce(counts[r:r + 1])
        return ev0, ev1

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    for r in range(args.warmup):
        device_round(r)
    barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tev = []
    with ClockSampler(local_rank) as clocks:
        barrier()
        t0.record()
        for r in range(args.warmup, total_rounds):
            tev.append(device_round(r))
        t1.record()
        barrier()
    ms = t0.elapsed_time(t1)
    train_ms = float(np.mean([a.elapsed_time(b) for a, b in tev]))
    if dist is not None:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    total_steps = args.steps * n_part * steps_per_client
    value = total_steps / (ms / 1e3)
    acc_last = counts[-1].item() / n_test

    # ---- e2e: public API per round (selection, DES, host PCG64 plan + H2D, train, FedAvg, D2H accuracy) ----
    def e2e_round(r, now):
        rep, mine, wl, seeds, _ = plan_round(r, now)
        fed.train(params, mine, wl, lr, seeds, deltas=deltas)
        if world == 1:
            fed.aggregate(params, deltas, [float(w.num_samples) for w in wl])
        else:
            aggregate(coef_of(mine))
        c = fed.correct(params)
        return now + rep.makespan, c

    now = 0.0
    for r in range(args.warmup):
        now, _ = e2e_round(total_rounds + r, now)
    barrier()
    e0 = time.perf_counter()
    for r in range(args.steps):
        now, c_last = e2e_round(total_rounds + args.warmup + r, now)
    barrier()
    e2e_s = time.perf_counter() - e0
    if dist is not None:
        t = torch.tensor([e2e_s], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    h2d = fed.last_h2d_bytes + per_gpu * 8     # permutations + descriptors, FedAvg coefficients

    flops = cnn_flop_per_sample(nc) * per_gpu * n_samp
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        peak, src = float(peaks["bf16_tflops"]), "MEASURED_PEAKS.json bf16_tflops (cuBLAS, measured)"
    except (OSError, KeyError, ValueError):
        peak, src = 1590.0, "fallback 1.59 PFLOP/s (B200_PROFILING.md)"
    tf = flops / (train_ms * 1e-3) / 1e12
    from benchlib import hbm_peak
    hbm_peak_v, hbm_src = hbm_peak(ROOT)
    p_canon = fed.layout.canonical_count
    hbm_alg = float(per_gpu * steps_per_client * (8 * p_canon + bs * (784 * 4 + 4)))
    n_launch = fed.engine.launches_per_round(steps_per_client)
    res = {
        "metric": "client local-steps/sec (FedHC round: local SGD of all participants + FedAvg + accuracy)",
        "value": value, "unit": "client-steps/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic, generated in HBM (Gaussian class clusters, Dirichlet(0.5) label mix); "
                                 "random-init FEMNIST CNN",
        "config": {"workload": f"femnist-cnn-c{nc}: BASELINE config 2, LEAF FEMNIST CNN clients "
                               f"(conv5x5 32, conv5x5 64, fc 2048, fc {nc})",
                   "arithmetic": "bf16 tensor-core operands (tcgen05), fp32 accumulation and fp32 master weights, "
                                 "FedAvg in fp64",
                   "participants_per_round": n_part, "fleet": n_fleet, "samples_per_client": n_samp, "batch": bs,
                   "local_steps_per_client": steps_per_client, "budgets": "10..100 step 10", "theta": THETA,
                   "scheduler": "resource-aware, dynamic parallelism", "max_executors": EXECUTORS,
                   "parallelism": f"clients sharded over {world} GPU(s)",
                   "l2": "per-client activations and weights (~4 GB/round) exceed L2; no flush needed"},
        "rounds_per_sec": args.steps / (ms / 1e3), "train_ms": train_ms, "accuracy_last_round": acc_last,
        "e2e": {"value": total_steps / e2e_s, "unit": "client-steps/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": 8, "rounds_per_sec": args.steps / e2e_s,
                "api": "CnnFederation.train / aggregate / correct (host selection, DES, PCG64 plan, H2D, D2H)"},
        # one SGD step streams every client's fp32 master weights in and out (8 B / param, the
        # algorithmic minimum of per-client SGD; AI = 123 flop/B < the 260 flop/B ridge): HBM-bound
        "roofline": {"bound": "hbm", "achieved": hbm_alg / (train_ms * 1e-3) / 1e9, "peak": hbm_peak_v,
                     "unit": "GB/s", "frac": hbm_alg / (train_ms * 1e-3) / 1e9 / hbm_peak_v, "traffic": None,
                     "kernel": "train phase (one CUDA graph: grouped_gemm_kernel launches incl. implicit-GEMM "
                               "conv2 + conv1/pool/CE kernels)",
                     "algorithmic_bytes_per_launch": hbm_alg,
                     "bytes_per_client_step": "8 x params (fp32 master read + write) + B x (784 x 4 + 4) input",
                     "peak_source": hbm_src},
        "roofline_tensor": {"bound": "tensor", "achieved": tf, "peak": peak, "unit": "TFLOP/s", "frac": tf / peak,
                            "algorithmic_flop_per_launch": flops, "flop_per_sample": cnn_flop_per_sample(nc),
                            "peak_source": src},
        "clocks": clocks.summary(),
        "gpu_launches": args.steps * (n_launch + 2 + (1 if world > 1 else 0)),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, cores, sample, _, _ = cnn_cpu_reference(args.cpu_seconds, nc, bs)
        res["cpu_baseline"] = {"value": v, "unit": "client-steps/s", "cores": cores, "kind": "port",
                               "sample": sample}
    if dist is not None:
        dist.destroy_process_group()
    return res


RESNET_FLOP_PER_SAMPLE = 3.329e9  # CIFAR ResNet-18 fwd + wgrad + dgrad (no stem dgrad), SURVEY §8a a14


def resnet_flop_per_sample(n_classes: int) -> float:
    """Algorithmic FLOPs of one training sample: 3 x forward convolutions minus the stem's data gradient."""
    macs, stem = 0, 32 * 32 * 64 * 27
    for ci, co, s, H in [(64, 64, 1, 32), (64, 64, 1, 32), (64, 128, 2, 32), (128, 128, 1, 16), (128, 256, 2, 16),
                         (256, 256, 1, 8), (256, 512, 2, 8), (512, 512, 1, 4)]:
        ho = H // s
        macs += ho * ho * co * 9 * ci + ho * ho * co * 9 * co + (ho * ho * co * ci if (s != 1 or ci != co) else 0)
    macs_fc = 512 * n_classes
    return float(2 * (3 * (macs + macs_fc) + 2 * stem))


def mobilenet_flop_per_sample(n_classes: int) -> float:
    """Algorithmic FLOPs of one MobileNetV2 training sample: 3 x forward (pointwise + depthwise + head +
    classifier) minus the stem's data gradient (unpadded channel counts)."""
    from paper_2305_15668_b200.mobilenet import HEAD, blocks
    macs, H, stem = 0, 32, 32 * 32 * 32 * 27
    for ci, pl, co, s in blocks():
        ho = H // s
        macs += H * H * ci * pl + ho * ho * pl * 9 + ho * ho * pl * co + (H * H * ci * co if s == 1 and ci != co else 0)
        H = ho
    macs += 16 * 320 * HEAD + HEAD * n_classes
    return float(2 * (3 * macs + 2 * stem))


def mobilenet_bytes_per_sample() -> float:
    """HBM roofline of the unfused MobileNetV2 layer graph, per training sample: every activation the
    backward needs (stem conv/BN-ReLU outputs; per block the expand output e and its BN-ReLU ea, the
    depthwise output d and da, the projection p, the shortcut conv output, the block output y; head conv
    output and its BN-ReLU) is written once and read once in bf16, and so is its gradient: 4 x 2 B per
    element, logical (unpadded) channel counts."""
    from paper_2305_15668_b200.mobilenet import HEAD, blocks
    el, H = 2 * 32 * 32 * 32, 32
    for ci, pl, co, s in blocks():
        ho = H // s
        el += 2 * H * H * pl + 2 * ho * ho * pl + 2 * ho * ho * co + (ho * ho * co if s == 1 and ci != co else 0)
        H = ho
    el += 2 * 16 * HEAD
    return float(4 * 2 * el)


def shufflenet_flop_per_sample(n_classes: int) -> float:
    """Algorithmic FLOPs of one ShuffleNetV2 x1.0 training sample (3 x forward minus the stem's data gradient)."""
    from paper_2305_15668_b200.shufflenet import HEAD, STAGES
    stem = 32 * 32 * 24 * 27
    macs = stem
    for cin, cout, nb, H in STAGES:
        mid, ho2 = cout // 2, (H // 2) ** 2
        macs += ho2 * cin * 9 + ho2 * cin * mid + H * H * cin * mid + ho2 * mid * 9 + ho2 * mid * mid
        macs += nb * (2 * ho2 * mid * mid + ho2 * mid * 9)
    macs += 16 * STAGES[2][1] * HEAD + HEAD * n_classes
    return float(2 * (3 * macs - stem))


def shufflenet_bytes_per_sample() -> float:
    """HBM roofline of the unfused ShuffleNetV2 layer graph per sample (as mobilenet_bytes_per_sample)."""
    from paper_2305_15668_b200.shufflenet import HEAD, STAGES
    el = 2 * 32 * 32 * 24
    for cin, cout, nb, H in STAGES:
        mid, ho2 = cout // 2, (H // 2) ** 2
        el += 2 * ho2 * cin + 2 * ho2 * mid + 2 * H * H * mid + 4 * ho2 * mid + ho2 * cout
        el += nb * (6 * ho2 * mid + ho2 * cout)
    el += 2 * 16 * HEAD
    return float(4 * 2 * el)


def cifar_cpu_reference(seconds: float, n_classes: int, batch: int, model: str = "resnet"):
    """CIFAR-model local SGD on the host cores (torch CPU, all threads): CPU restatement (no reference CNN)."""
    import torch
    import torch.nn as nn

    if model == "mobilenet":
        from oracle.mobilenet import MobileNetV2 as Net
        name = "MobileNetV2"
    elif model == "shufflenet":
        from oracle.shufflenet import ShuffleNetV2 as Net
        name = "ShuffleNetV2"
    else:
        from oracle.resnet import ResNet18 as Net
        name = "ResNet-18"
    cores = len(os.sched_getaffinity(0))
    torch.set_num_threads(cores)
    torch.manual_seed(0)
    net = Net(n_classes)
    net.train()
    opt = torch.optim.SGD(net.parameters(), lr=0.05)
    x = torch.randn(256, 3, 32, 32)
    y = torch.randint(0, n_classes, (256,))
    lossf = nn.CrossEntropyLoss()

    def one(i):
        s0 = (i * batch) % (256 - batch)
        opt.zero_grad(set_to_none=True)
        lossf(net(x[s0:s0 + batch]), y[s0:s0 + batch]).backward()
        opt.step()

    for i in range(2):
        one(i)
    n, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < seconds:
        one(n)
        n += 1
    dt = time.perf_counter() - t0
    return n / dt, cores, (f"{n} local SGD steps (B={batch}) of one {name} client, torch CPU fp32 with {cores} "
                           f"threads (CPU restatement: the reference has no CNN)"), n, dt


def run_resnet(args, rank, world, local_rank, model="resnet"):
    """BASELINE config 3 with its named model: CIFAR ResNet-18 clients, 200 participants per round sharded
    over the GPUs (25 per GPU at 8 GPUs; --resnet-clients per GPU), 250 samples each, B = 32.
    model="mobilenet": BASELINE config 4 -- CIFAR MobileNetV2 clients from a fleet of >= 1000 with non-IID
    sample counts (uniform choice of 16, 32, ..., 1024), --mobilenet-clients participants per GPU, B = 32;
    each local step runs only the clients that still have batches (clients in descending-step order)."""
    import torch

    import paper_2305_15668_b200 as fh
    from paper_2305_15668_b200.devicedata import DeviceFleetData
    from paper_2305_15668_b200.experiment import delta_buffer
    if model == "mobilenet":
        from paper_2305_15668_b200.mobilenet import MobilenetFederation as Federation
        from paper_2305_15668_b200.mobilenet import init_mobilenet_params as init_params
    elif model == "shufflenet":
        from paper_2305_15668_b200.shufflenet import ShufflenetFederation as Federation
        from paper_2305_15668_b200.shufflenet import init_shufflenet_params as init_params
    else:
        from paper_2305_15668_b200.resnet import ResnetFederation as Federation
        from paper_2305_15668_b200.resnet import init_resnet_params as init_params
    from paper_2305_15668_b200.roundsim import RoundSimulator
    from paper_2305_15668_b200.sharding import shard_bounds
    from paper_2305_15668_b200.training import fedavg_device, stable_seed

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist_mod
        dist = dist_mod
        dist.init_process_group("nccl", device_id=dev)
    nc, bs, lr = 10, 32, 0.05
    config4 = model in ("mobilenet", "shufflenet")
    if config4:
        per_gpu = args.mobilenet_clients
        n_part, n_fleet = per_gpu * world, max(args.mobilenet_fleet, per_gpu * world)
        levels, v = [], 16
        while v <= args.mobilenet_max_samples:
            levels.append(v)
            v *= 2
        n_samp = levels
    else:
        n_samp = args.resnet_samples
        per_gpu = args.resnet_clients
        n_part, n_fleet = per_gpu * world, (per_gpu + per_gpu // 4) * world
    if args.strong:  # config 3: a fixed round (e.g. 200 participants) split over the ranks
        n_part = args.resnet_total
        n_fleet = max(n_fleet, n_part + n_part // 4) if not config4 else max(args.mobilenet_fleet, n_part)
    fleet = fh.generate_fleet(fh.DistributionSpec(budget_levels=BUDGETS, num_samples=n_samp, batch_size=bs),
                              n_fleet, 3)
    by_id = {p.client_id: p for p in fleet}
    ids = sorted(by_id)
    from paper_2305_15668_b200.sharding import client_cost, lpt_shards
    total_rounds = args.warmup + args.steps

    def my_share(who):
        """LPT shard of the round's selection for this rank (rows processed per client), selection order."""
        costs = [client_cost(by_id[c].workload.num_samples, bs) for c in who]
        return [who[j] for j in lpt_shards(costs, world)[rank]]

    # engine capacity = the largest share this rank gets in any round (device-resident + e2e rounds)
    _sel = random.Random("3:selection")
    per_gpu = max(len(my_share(_sel.sample(ids, n_part))) for _ in range(2 * total_rounds + args.warmup))
    n_test = 2048
    data = DeviceFleetData(ids, [by_id[c].workload.num_samples for c in ids], 3072, nc, alpha=0.5, seed=4321,
                           n_test=n_test)
    lo, hi = shard_bounds(n_test, world, rank)
    fed = Federation.from_arrays(data.x, data.y, data.offsets, data.x_test[lo:hi].contiguous(),
                                       data.y_test[lo:hi].contiguous(), nc).attach_engine(per_gpu, bs)
    P = fed.P
    params = torch.tensor(fed.layout.to_padded(init_params(nc, 1)), dtype=torch.float64, device=dev)
    deltas = delta_buffer(per_gpu, P, dev)
    partial = torch.empty(P, dtype=torch.float64, device=dev)
    one = torch.ones(1, dtype=torch.float64, device=dev)
    cfg = fh.FleetConfig(theta=THETA, max_executors=EXECUTORS, participants_per_round=n_part, seed=3)
    sim = RoundSimulator(by_id)
    selector = random.Random(f"{cfg.seed}:selection")

    def plan_round(r, now):
        who = selector.sample(ids, n_part)
        rep, _ = sim.run(who, cfg, t0=now, round_index=r, want_trace=False)
        mine = my_share(who)
        wl = [by_id[c].workload for c in mine]
        seeds = [stable_seed("train", cfg.seed, r, c) for c in mine]
        tot = float(sum(float(by_id[c].workload.num_samples) for c in who))  # W over the whole round
        coef = torch.tensor([float(w.num_samples) / tot for w in wl], dtype=torch.float64, device=dev)
        return rep, mine, wl, seeds, coef

    def aggregate(coef, k=None):
        k = coef.shape[0] if k is None else k
        if world == 1:
            fedavg_device(deltas[:k], coef, params, params)
        else:
            if k:
                fedavg_device(deltas[:k], coef, None, partial)
            else:
                partial.zero_()
            dist.all_reduce(partial)
            fedavg_device(partial.view(1, -1), one, params, params)

    plans, now = [], 0.0
    for r in range(total_rounds):
        rep, mine, wl, seeds, coef = plan_round(r, now)
        now += rep.makespan
        packed, meta = fed.plan(mine, wl, seeds)
        perm_dev = torch.from_numpy(packed).to(dev)
        fed._perm_dev = perm_dev
        order = sorted(range(len(mine)), key=lambda i: -meta[i][2])  # descending local steps
        desc = fed.descriptors([mine[i] for i in order], [meta[i] for i in order], lr, deltas, rows=order)
        steps = [meta[i][2] for i in order]
        plans.append((perm_dev, desc, coef, steps, sum(steps), sum(w.num_samples for w in wl)))
    counts = torch.zeros(total_rounds, dtype=torch.int64, device=dev)

    def device_round(r):
        _, desc, coef, steps, _, _ = plans[r]
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        if config4:
            fed.engine.local_train(desc.data_ptr(), len(steps), params, steps[0], lr, True, steps=steps)
        else:
            fed.engine.local_train(desc.data_ptr(), len(steps), params, steps[0], lr, True)
        ev1.record()
        aggregate(coef)
        fed.engine.correct_into(params, fed.x_test, fed.y_test, counts[r:r + 1])
        if world > 1:
            dist.all_reduce(counts[r:r + 1])
        return ev0, ev1

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    for r in range(args.warmup):
        device_round(r)
    barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tev = []
    lc0 = fed.engine.launch_count()
    with ClockSampler(local_rank) as clocks:
        barrier()
        t0.record()
        for r in range(args.warmup, total_rounds):
            tev.append(device_round(r))
        t1.record()
        barrier()
    ms = t0.elapsed_time(t1)
    # our kernels in the timed region: engine graph nodes + direct launches (train, eval) + FedAvg (1, or 2 with
    # the all-reduce split)
    launches = fed.engine.launch_count() - lc0 + args.steps * (1 if world == 1 else 2)
    train_ms = float(np.mean([a.elapsed_time(b) for a, b in tev]))
    if dist is not None:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    timed = plans[args.warmup:]
    total_steps = sum(p[4] for p in timed)  # client local steps of this GPU's clients, then of all GPUs
    if dist is not None:
        t = torch.tensor([total_steps], dtype=torch.int64, device=dev)
        dist.all_reduce(t)
        total_steps = int(t.item())
    value = total_steps / (ms / 1e3)

    # e2e: public API per round (selection, DES, host PCG64 plan + H2D, train, FedAvg, D2H accuracy)
    e2e_counts = []

    def e2e_round(r, now, count=False):
        rep, mine, wl, seeds, coef = plan_round(r, now)
        if count:
            e2e_counts.append(sum(math.ceil(w.num_samples / bs) for w in wl))
        fed.train(params, mine, wl, lr, seeds, deltas=deltas)
        if world == 1:
            fed.aggregate(params, deltas, [float(w.num_samples) for w in wl])
        else:
            aggregate(coef, len(mine))
        fed.correct(params)
        return now + rep.makespan

    now = 0.0
    for r in range(args.warmup):
        now = e2e_round(total_rounds + r, now)
    barrier()
    e0 = time.perf_counter()
    for r in range(args.steps):
        now = e2e_round(total_rounds + args.warmup + r, now, count=True)
    barrier()
    e2e_s = time.perf_counter() - e0
    e2e_steps = sum(e2e_counts)
    if dist is not None:
        t = torch.tensor([e2e_s], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
        t = torch.tensor([e2e_steps], dtype=torch.int64, device=dev)
        dist.all_reduce(t)
        e2e_steps = int(t.item())

    fps = (mobilenet_flop_per_sample(nc) if model == "mobilenet" else shufflenet_flop_per_sample(nc)
           if model == "shufflenet" else resnet_flop_per_sample(nc))
    flops = fps * float(np.mean([p[5] for p in timed]))  # per train launch (this GPU's samples)
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        peak, src = float(peaks["bf16_tflops"]), "MEASURED_PEAKS.json bf16_tflops (cuBLAS, measured)"
    except (OSError, KeyError, ValueError):
        peak, src = 1590.0, "fallback 1.59 PFLOP/s (B200_PROFILING.md)"
    tf = flops / (train_ms * 1e-3) / 1e12
    hbm_roof = None
    if config4:
        try:
            hpk, hsrc = float(peaks["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy, measured)"
        except (NameError, KeyError, ValueError):
            hpk, hsrc = 6543.7, "fallback 6.54 TB/s (SURVEY §8d)"
        p_canon = fed.layout.canonical_count
        steps_round = float(np.mean([p[4] for p in timed]))
        bps_ = mobilenet_bytes_per_sample() if model == "mobilenet" else shufflenet_bytes_per_sample()
        bytes_launch = bps_ * float(np.mean([p[5] for p in timed])) + 8.0 * p_canon * steps_round
        gbs = bytes_launch / (train_ms * 1e-3) / 1e9
        hbm_roof = {"bound": "hbm", "achieved": gbs, "peak": hpk, "unit": "GB/s", "frac": gbs / hpk, "traffic": None,
                    "kernel": "train phase (see roofline_tensor for the kernels)",
                    "algorithmic_bytes_per_launch": bytes_launch,
                    "bytes_per_sample": bps_, "weight_bytes_per_client_step": 8.0 * p_canon,
                    "peak_source": hsrc,
                    "note": f"arithmetic intensity {fps / bps_:.0f} flop/B << ridge (~260): HBM-bound"}
    if model == "shufflenet":
        mname, cfg_name = "ShuffleNetV2", ("cifar-shufflenetv2: BASELINE config 4 model, ShuffleNetV2 x1.0 (CIFAR "
                                           "variant: 3x3 stem, stages 116-232-464 with channel split / shuffle, "
                                           "1x1 head to 1024, batch norm), 10 classes, fleet of %d with non-IID "
                                           "sample counts" % n_fleet)
        api = "ShufflenetFederation.train / aggregate / correct (host selection, DES, PCG64 plan, H2D, D2H)"
        kern = ("train phase (one CUDA graph per active-client count: 1x1 convolutions as grouped tcgen05 GEMMs with "
                "strided split-form operands, depthwise 3x3 kernels, shuffle / BN kernels)")
        spc = "ceil(n / 32) for n in " + str(n_samp)
        arith = ("bf16 tensor-core operands and activations (tcgen05) for the 1x1 convolutions, FHFMA depthwise "
                 "3x3, fp32 accumulation, batch norm and master weights; FedAvg in fp64")
    elif model == "mobilenet":
        mname, cfg_name = "MobileNetV2", ("cifar-mobilenetv2: BASELINE config 4 model, MobileNetV2 (CIFAR variant: "
                                           "3x3 stem, 17 inverted-residual blocks, 1x1 head to 1280, batch norm), "
                                           "10 classes, fleet of %d with non-IID sample counts" % n_fleet)
        api = "MobilenetFederation.train / aggregate / correct (host selection, DES, PCG64 plan, H2D, D2H)"
        kern = ("train phase (one CUDA graph per active-client count: pointwise convolutions as implicit-GEMM "
                "grouped_gemm_kernel launches, depthwise 3x3 CUDA-core kernels, batch-norm / elementwise kernels)")
        spc = "ceil(n / 32) for n in " + str(n_samp)
        arith = ("bf16 tensor-core operands and activations (tcgen05) for the pointwise / head convolutions, fp32 "
                 "CUDA-core depthwise 3x3 on bf16 activations, fp32 accumulation, batch norm and master weights; "
                 "FedAvg in fp64")
    else:
        mname, cfg_name = "ResNet-18", ("cifar-resnet18: BASELINE config 3 model, ResNet-18 (3x3 stem, BasicBlocks "
                                        "64-128-256-512, batch norm), 10 classes")
        api = "ResnetFederation.train / aggregate / correct (host selection, DES, PCG64 plan, H2D, D2H)"
        kern = ("train phase (one CUDA graph: implicit-GEMM grouped_gemm_kernel launches + batch-norm / "
                "elementwise kernels)")
        spc = math.ceil(n_samp / bs)
        arith = ("bf16 tensor-core operands and activations (tcgen05), fp32 accumulation, batch norm and master "
                 "weights; FedAvg in fp64")
    res = {
        "metric": "client local-steps/sec (FedHC round: local SGD of all participants + FedAvg + accuracy)",
        "value": value, "unit": "client-steps/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong" if args.strong else "weak",
        "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic CIFAR-shaped 32x32x3 rows generated in HBM (Gaussian class clusters, "
                                 "Dirichlet(0.5) label mix); random-init " + mname,
        "config": {"workload": cfg_name, "arithmetic": arith,
                   "participants_per_round": n_part, "per_gpu": per_gpu, "fleet": n_fleet,
                   "samples_per_client": n_samp, "batch": bs, "local_steps_per_client": spc,
                   "budgets": "10..100 step 10", "theta": THETA, "scheduler": "resource-aware, dynamic parallelism",
                   "parallelism": f"clients LPT-sharded over {world} GPU(s) ({per_gpu} max per GPU)"
                                  + (", NCCL all-reduce of FedAvg partials" if world > 1 else ""),
                   "l2": "per-client weights + activations (GBs per round) exceed L2; no flush needed"},
        "rounds_per_sec": args.steps / (ms / 1e3), "train_ms": train_ms,
        "client_steps_per_round": total_steps / args.steps,
        "accuracy_last_round": counts[-1].item() / n_test,
        "e2e": {"value": e2e_steps / e2e_s, "unit": "client-steps/s",
                "h2d_bytes_per_step": int(fed.last_h2d_bytes + per_gpu * 8), "d2h_bytes_per_step": 8,
                "rounds_per_sec": args.steps / e2e_s, "api": api},
        "roofline": hbm_roof or {"bound": "tensor", "achieved": tf, "peak": peak, "unit": "TFLOP/s",
                                 "frac": tf / peak, "traffic": None, "kernel": kern,
                                 "algorithmic_flop_per_launch": flops, "flop_per_sample": fps, "peak_source": src},
        "roofline_tensor": {"bound": "tensor", "achieved": tf, "peak": peak, "unit": "TFLOP/s", "frac": tf / peak,
                            "kernel": kern, "algorithmic_flop_per_launch": flops, "flop_per_sample": fps,
                            "peak_source": src},
        "clocks": clocks.summary(),
        "gpu_launches": launches,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, cores, sample, _, _ = cifar_cpu_reference(args.cpu_seconds, nc, bs, model)
        res["cpu_baseline"] = {"value": v, "unit": "client-steps/s", "cores": cores, "kind": "port", "sample": sample}
    if dist is not None:
        dist.destroy_process_group()
    return res


def run_reference(args, rank, world):
    """--impl reference: the reference algorithm's CPU implementation (oracle port), rank 0 only."""
    if rank != 0:
        return None
    if args.workload in ("cnn", "resnet", "mobilenet", "shufflenet"):
        # the reference has no CNN: its arm for the CNN workloads is the torch-CPU restatement of the same
        # client step (the CPU baseline of those workloads), on all host threads
        if args.workload == "cnn":
            v, cores, sample, _, secs = cnn_cpu_reference(args.cpu_seconds, args.classes, 64)
        else:
            v, cores, sample, _, secs = cifar_cpu_reference(args.cpu_seconds, 10, 32, args.workload)
        return {
            "impl": "reference", "metric": "client local-steps/sec (FedHC round: local SGD of all participants + "
                                           "FedAvg + accuracy)",
            "value": v, "unit": "client-steps/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 / v if v else None, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{args.workload}: torch-CPU restatement of one client's local SGD step"},
            "cpu_baseline": {"value": v, "unit": "client-steps/s", "cores": cores, "kind": "port", "sample": sample},
            "e2e": {"value": v, "unit": "client-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }
    v, cores, sample, rounds, secs = cpu_reference(0.0, rounds=args.steps, warmup=args.warmup)
    return {
        "impl": "reference",
        "metric": "client local-steps/sec (FedHC round: local SGD of all participants + FedAvg + accuracy)",
        "value": v,
        "unit": "client-steps/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": secs / max(rounds, 1) * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": workload_config(1),
        "cpu_baseline": {"value": v, "unit": "client-steps/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": v, "unit": "client-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def _relaunch_under_torchrun(n: int) -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    global C
    args = parse()
    C = args.classes
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # launched without torchrun: spawn one rank per GPU ourselves (same contract as the driver's
        # `torch.distributed.run --nproc-per-node N ... bench.py --gpus N`), rank 0 prints the line
        sys.exit(_relaunch_under_torchrun(args.gpus))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(1)))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one rank per GPU "
                         f"(torchrun --nproc-per-node {args.gpus}) or omit torchrun\n")
        sys.exit(2)
    if args.impl == "reference":
        res = run_reference(args, rank, world)
    elif args.workload == "fedavg":
        res = run_fedavg(args, rank, world, local_rank)
    elif args.workload == "cnn":
        res = run_cnn(args, rank, world, local_rank)
    elif args.workload == "resnet":
        res = run_resnet(args, rank, world, local_rank)
    elif args.workload == "mobilenet":
        res = run_resnet(args, rank, world, local_rank, model="mobilenet")
    elif args.workload == "shufflenet":
        res = run_resnet(args, rank, world, local_rank, model="shufflenet")
    elif args.workload == "gemm":
        res = run_gemm(args, rank, world, local_rank)
    elif args.workload == "live":
        res = run_live(args, rank, world, local_rank)
    elif args.workload == "des":
        res = run_des(args) if rank == 0 else None
    elif args.workload == "data":
        res = run_data(args, local_rank) if rank == 0 else None
    else:
        res = run_ours(args, rank, world, local_rank)
    if rank == 0 and res is not None:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
