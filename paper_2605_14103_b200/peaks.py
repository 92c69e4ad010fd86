"""Roofline denominators: MEASURED_PEAKS.json (driver-written) + our FP64 probe."""

from __future__ import annotations

import json
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
# profiles/r2/fp64_peak_r2_clocks.txt: DMMA m8n8k4 best configuration, 5 runs at
# 1965 MHz (clock record alongside; r1: profiles/fp64_peak_r1.txt, same value)
FP64_DMMA_TFLOPS = 37.09
FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback


def hbm_gbs() -> tuple:
    try:
        d = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def fp64_tflops() -> tuple:
    return FP64_DMMA_TFLOPS, "measured DMMA f64 at 1965 MHz (profiles/r2/fp64_peak_r2_clocks.txt)"
