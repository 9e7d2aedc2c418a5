"""Helpers shared by the bench legs: peaks, clocks, CPU thread count."""
from __future__ import annotations

import json
import os

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def peaks():
    """(bf16 sustained TFLOP/s, bf16 burst TFLOP/s, HBM GB/s, source)."""
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return d["bf16_tflops_sustained"], d["bf16_tflops"], d["hbm_gbs"], "measured"
    except Exception:
        return 1400.0, 1590.0, 6650.0, "fallback"


def ncu_traffic(kernel):
    try:
        with open(os.path.join(REPO, "profiles", "ncu_summary.json")) as f:
            return json.load(f).get(kernel, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1
