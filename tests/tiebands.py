"""Stop-rule tie-band classifier (SURVEY.md §0 fact 9, §7 hard part 5).

The Z-Bus loop stops at the first sweep k with
delta_k = |sum|v_k| - sum|v_k-1|| <= tol (reference distribution.py:674-679);
Newton stops at the first check with ||F||inf <= tol (transmission.py:353).
The engine sums in a different (fixed) order than numpy, so a scenario whose
reference decision value sits within rounding of tol may stop one step
earlier or later. Such a mismatch is a TIE, never hidden: it is reported
separately and only tolerated when the reference's own margin
|delta_ref - tol| at the deciding step is below `band` * tol.
"""

from __future__ import annotations

import numpy as np

BAND = 1e-3  # relative tie band: |delta_ref - tol| < 1e-3 * tol


def classify(ref_iters, got_iters, ref_decision, tol: float, band: float = BAND, first: int = 1):
    """Split iteration-count mismatches into ties and real mismatches.

    ref_decision[s, j] is the reference's decision value at step j + first
    (Z-Bus: sweep j+1's delta, first = 1; Newton: the check at k = j,
    first = 0), NaN past the reference's exit. For a mismatch the deciding
    step is min(ref, got): at that step one side stopped and the other did not,
    so the reference's value there must lie within the band of tol.
    Returns (ties, real): index arrays.
    """
    ref_iters = np.asarray(ref_iters)
    got_iters = np.asarray(got_iters)
    bad = np.flatnonzero(ref_iters != got_iters)
    ties, real = [], []
    for s in bad:
        k = int(min(ref_iters[s], got_iters[s])) - first
        row = ref_decision[s]
        val = row[k] if 0 <= k < row.size else np.nan
        (ties if np.isfinite(val) and abs(val - tol) < band * tol else real).append(int(s))
    return np.array(ties, dtype=np.int64), np.array(real, dtype=np.int64)


def margins(ref_iters, ref_decision, tol: float, first: int = 1):
    """Smallest relative distance of any scenario's stop decision to tol: at the
    stopping step (value <= tol) and at the step before (value > tol)."""
    ref_iters = np.asarray(ref_iters)
    m = np.inf
    for s in range(ref_iters.size):
        k = int(ref_iters[s]) - first
        row = ref_decision[s]
        for j in (k - 1, k):
            if 0 <= j < row.size and np.isfinite(row[j]):
                m = min(m, abs(row[j] - tol) / tol)
    return m


def report(name: str, ties, real, n: int) -> str:
    return f"{name}: {n} scenarios, {ties.size} stop-rule ties (reported), {real.size} real mismatches"


def check_iterations(name: str, ref_iters, got_iters, ref_decision, tol: float, first: int):
    """Assert every iteration-count mismatch is a stop-rule tie; return the tie
    indices (report them, exclude them from state comparisons). The report
    line goes to stdout and, if ACPF_TIE_REPORT names a file, is appended there."""
    import os

    ties, real = classify(ref_iters, got_iters, ref_decision, tol, first=first)
    line = (report(name, ties, real, len(ref_iters))
            + f"; reference min stop margin {margins(ref_iters, ref_decision, tol, first):.3e} x tol"
            + (f"; tie rows {ties.tolist()[:20]}" if ties.size else ""))
    print(line)
    path = os.environ.get("ACPF_TIE_REPORT")
    if path:
        with open(path, "a") as fh:
            fh.write(line + "\n")
    assert real.size == 0, f"{name}: non-tie iteration mismatches at {real.tolist()[:20]}"
    return ties
