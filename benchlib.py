"""Helpers for bench.py: roofline bookkeeping against MEASURED_PEAKS.json."""

from __future__ import annotations

import json
import os

FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback


def hbm_peak(root: str):
    path = os.path.join(root, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy)"
    except (OSError, KeyError, ValueError):
        return FALLBACK_HBM_GBS, "fallback 6.65 TB/s (B200_PROFILING.md)"


def profiled_traffic(root: str, kernel: str):
    """dram bytes per launch from the committed ncu --set full summary, if present."""
    path = os.path.join(root, "profiles", "traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh).get(kernel)
    except (OSError, ValueError):
        return None


def roofline_entry(bytes_per_launch: float, launch_ms: float, root: str, kernel: str = "train_fused_kernel"):
    peak, src = hbm_peak(root)
    achieved = bytes_per_launch / (launch_ms * 1e-3) / 1e9
    return {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": profiled_traffic(root, kernel), "kernel": kernel,
            "algorithmic_bytes_per_launch": bytes_per_launch, "peak_source": src}
