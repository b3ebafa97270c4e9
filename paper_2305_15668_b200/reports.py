"""Experiment output files in the reference's formats.

Same names, columns, number formatting and key order as fedsim's `simulate`
writers (cli.py:38-102, pkg/docs/schemas.md): trace.jsonl, rounds.csv,
clients.csv, summary.json, fleet.csv.  Simulated times come from the native
DES (bit-identical to the reference), so these files are byte-identical to
the reference's for the same configuration whenever training is disabled;
with training, `accuracy_series` carries the GPU-trained accuracies.
"""

from __future__ import annotations

import csv
import json
import os
from dataclasses import asdict, is_dataclass

from .roundsim import write_trace_jsonl
from .spec import save_fleet

_G = "{:.9g}".format


def write_rounds_csv(path, report) -> None:
    with open(path, "w", newline="") as fh:
        out = csv.writer(fh)
        out.writerow(["round", "makespan_s", "utilization", "vacancy_area", "throughput", "n_clients"])
        for r in report.rounds:
            d = r.to_dict()
            out.writerow([d["round"], _G(d["makespan_s"]), _G(d["utilization"]), _G(d["vacancy_area"]),
                          _G(d["throughput"]), d["n_clients"]])


def write_clients_csv(path, report) -> None:
    with open(path, "w", newline="") as fh:
        out = csv.writer(fh)
        out.writerow(["round", "client_id", "budget", "start_s", "end_s", "wall_clock_s"])
        for r in report.rounds:
            for cid in sorted(r.per_client_times):
                out.writerow([r.round_index, cid, _G(r.per_client_budget[cid]), _G(r.per_client_start[cid]),
                              _G(r.per_client_end[cid]), _G(r.per_client_times[cid])])


def write_summary(path, report, config=None) -> None:
    if is_dataclass(config):
        config = asdict(config)
    payload = {
        "config": config if config is not None else {},
        "rounds": [r.to_dict() for r in report.rounds],
        "participants": report.participants,
        "accuracy_series": report.accuracy_series,
        "total_time": report.total_time,
        "mean_round_time": report.mean_round_time(),
    }
    with open(path, "w") as fh:
        json.dump(payload, fh, sort_keys=True, indent=2)
        fh.write("\n")


def write_outputs(out_dir, report, trace=None, fleet=None, config=None) -> str:
    """Write every `simulate` output into out_dir (FEDSIM_OUT overrides, as in cli.py:32-35)."""
    out_dir = os.environ.get("FEDSIM_OUT", out_dir)
    os.makedirs(out_dir, exist_ok=True)
    if trace is not None:
        write_trace_jsonl(trace, os.path.join(out_dir, "trace.jsonl"))
    write_rounds_csv(os.path.join(out_dir, "rounds.csv"), report)
    write_clients_csv(os.path.join(out_dir, "clients.csv"), report)
    write_summary(os.path.join(out_dir, "summary.json"), report, config)
    if fleet is not None:
        save_fleet(fleet, os.path.join(out_dir, "fleet.csv"))
    return out_dir
