"""Array-backed scenario batches and results, and the multi-device solve.

The reference's batched API moves one Python object per scenario
(``make_scenarios`` -> list of scenarios, ``run_batch`` / ``batch_zbus_solve``
-> list of results; batch.py:154-159, :280-344, distribution.py:690-711). At
10^5-10^6 scenarios that host work costs as much as the device solve, so this
package keeps both sides stacked:

* :class:`TransmissionScenarios` / :class:`DistributionScenarios` are
  sequences of scenario objects backed by the stacked input arrays the C-ABI
  consumes; items are created on first access (views, memoised so identity
  holds), and the solvers take the arrays without re-stacking.
* :class:`NewtonResults` / :class:`ZbusResults` are sequences of
  ``NewtonResult`` / ``FixedPointResult`` backed by the stacked outputs;
  ``run_batch`` builds its records from the arrays directly.

Per-scenario isolation (reference batch.py:237-239, distribution.py:714-727):
a malformed scenario (wrong shape, not numeric) never reaches the device and
never poisons the batch: it becomes a failed record carrying the error text,
exactly as the reference's ``_safe_zbus`` / ``_timed_solve`` record it.

Multi-device (replaces the reference's fork pool,
batch.py:204-217, :313-330): :func:`solve_sharded` splits the batch into
contiguous ranges, one per entry of ``devices`` (one plan per entry, so the
same device may appear twice), drives each plan from its own host thread
(ctypes releases the GIL for the C-ABI call; plans on different devices run
concurrently, include/acpf.h threading rules) and the library writes each
shard straight into its rows of the caller's output arrays, so the gather is
the output itself. No collective is involved.
"""

from __future__ import annotations

from collections.abc import Sequence
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from .shard import shard_range


def _failure(exc: BaseException) -> str:
    return f"{type(exc).__name__}: {exc}"


# ---------------------------------------------------------------------------
# scenario batches
# ---------------------------------------------------------------------------


class _StackedScenarios(Sequence):
    _fields: tuple = ()

    def __init__(self, *arrays):
        self._arrays = arrays
        self._items = [None] * int(arrays[0].shape[0])

    def __len__(self):
        return len(self._items)

    def __getitem__(self, k):
        if isinstance(k, slice):
            return [self[i] for i in range(*k.indices(len(self)))]
        if k < 0:
            k += len(self)
        it = self._items[k]
        if it is None:
            it = self._items[k] = self._make(*(a[k] for a in self._arrays))
        return it

    @property
    def arrays(self) -> tuple:
        return self._arrays


class TransmissionScenarios(_StackedScenarios):
    """Sequence of ``TransmissionScenario`` over stacked (p_spec[B, n_theta], q_spec[B, n_q])."""

    @staticmethod
    def _make(p, q):
        from .transmission import TransmissionScenario
        return TransmissionScenario(p_spec=p, q_spec=q)


class DistributionScenarios(_StackedScenarios):
    """Sequence of ``DistributionScenario`` over stacked (s_wye[B, n_wye], s_delta[B, n_delta])."""

    @staticmethod
    def _make(w, d):
        from .distribution import DistributionScenario
        return DistributionScenario(wye_s=w, delta_s=d)


def stack_checked(scenarios, fields: tuple, widths: tuple, dtype, batch_cls):
    """Stacked inputs for the valid scenarios plus {index: error} for the rest.

    A scenario is valid when every field converts to a 1-D array of the
    expected width and dtype; anything else is recorded as that scenario's
    error (the reference records a raising solve the same way)."""
    if isinstance(scenarios, batch_cls):
        arrs = scenarios.arrays
        if all(a.ndim == 2 and a.shape[1] == w for a, w in zip(arrs, widths)):
            return tuple(np.ascontiguousarray(a, dtype=dtype) for a in arrs), np.arange(len(scenarios)), {}
    n = len(scenarios)
    errors = {}
    ok = []
    rows = [[] for _ in fields]
    for k, sc in enumerate(scenarios):
        try:
            vals = []
            for f, w in zip(fields, widths):
                a = np.asarray(getattr(sc, f))
                if a.dtype.kind not in "biufc" or a.shape != (w,):
                    raise ValueError(f"scenario.{f} must be a numeric vector of length {w}, "
                                     f"got shape {a.shape} dtype {a.dtype}")
                if dtype != np.complex128 and a.dtype.kind == "c":
                    raise ValueError(f"scenario.{f} must be real")
                vals.append(a)
        except Exception as exc:  # isolate, never poison the batch
            errors[k] = _failure(exc)
            continue
        ok.append(k)
        for r, a in zip(rows, vals):
            r.append(a)
    out = []
    for r, w in zip(rows, widths):
        if r:
            out.append(np.ascontiguousarray(np.stack(r), dtype=dtype))
        else:
            out.append(np.empty((0, w), dtype=dtype))
    return tuple(out), np.asarray(ok, dtype=np.int64), errors


# ---------------------------------------------------------------------------
# results
# ---------------------------------------------------------------------------


class _Results(Sequence):
    """Sequence over stacked engine outputs; rows listed in ``errors`` failed
    before the device (their arrays rows hold the failed-record values)."""

    def __init__(self, out: dict, errors: dict | None = None):
        self.out = out
        self.errors = dict(errors or {})
        self._n = int(out["converged"].shape[0])

    def __len__(self):
        return self._n

    def __getitem__(self, k):
        if isinstance(k, slice):
            return [self[i] for i in range(*k.indices(len(self)))]
        if k < 0:
            k += self._n
        if not 0 <= k < self._n:
            raise IndexError(k)
        return self._item(k)

    def __eq__(self, other):
        return list(self) == list(other)

    # vectorised record fields (run_batch)
    def converged(self) -> np.ndarray:
        return self.out["converged"].astype(bool)

    def iterations(self) -> np.ndarray:
        return self.out["iterations"].astype(np.int64)


class NewtonResults(_Results):
    """``NewtonResult`` records over ``batch_newton_solve``'s stacked outputs."""

    def _item(self, k):
        from .transmission import NewtonResult, PolarState, status_diagnostic
        o = self.out
        it = int(o["iterations"][k])
        per = ()
        diag = None
        if k in self.errors:
            diag = self.errors[k]
        else:
            if "gmres_steps" in o:
                per = tuple(int(c) for c in o["gmres_steps"][k][:it])
            diag = status_diagnostic(o, k)
        return NewtonResult(state=PolarState(o["theta"][k], o["vmag"][k]), converged=bool(o["converged"][k]),
                            iterations=it, final_mismatch_inf=float(o["final_mismatch_inf"][k]),
                            per_iteration_gmres=per, diagnostic=diag)

    def residuals(self) -> np.ndarray:
        return np.asarray(self.out["final_mismatch_inf"], dtype=np.float64)

    def diagnostics(self) -> list:
        from .transmission import status_diagnostic
        st = self.out["status"]
        res = [None] * self._n
        for k in np.flatnonzero(st != 0):  # converged rows carry no diagnostic (LU step)
            res[k] = status_diagnostic(self.out, int(k))
        if "gmres_diag" in self.out:
            for k in np.flatnonzero(self.out["gmres_diag"] != 0):
                res[k] = status_diagnostic(self.out, int(k))
        for k, msg in self.errors.items():
            res[k] = msg
        return res


class ZbusResults(_Results):
    """``FixedPointResult`` records over ``batch_zbus_solve``'s stacked outputs."""

    def __init__(self, model, out: dict, errors: dict | None = None):
        super().__init__(out, errors)
        self.model = model

    def _item(self, k):
        from .distribution import FixedPointResult
        from .engine import ZB_FLOOR, zbus_floor_message
        o = self.out
        if k in self.errors:
            diag = self.errors[k]
        elif int(o["status"][k]) == ZB_FLOOR:
            diag = zbus_floor_message(self.model, o["v"][k], int(o["floor_slot"][k]))
        else:
            diag = None
        return FixedPointResult(v=o["v"][k], converged=bool(o["converged"][k]), iterations=int(o["iterations"][k]),
                                final_delta=float(o["final_delta"][k]), residual_inf=float(o["residual_inf"][k]),
                                diagnostic=diag)

    def residuals(self) -> np.ndarray:
        return np.asarray(self.out["residual_inf"], dtype=np.float64)

    def diagnostics(self) -> list:
        from .engine import ZB_FLOOR
        res = [None] * self._n
        for k in np.flatnonzero(self.out["status"] == ZB_FLOOR):
            res[k] = self._item(int(k)).diagnostic
        for k, msg in self.errors.items():
            res[k] = msg
        return res


def scatter_rows(out_valid: dict, idx: np.ndarray, n: int, fill: dict) -> dict:
    """Full-size outputs: valid rows from ``out_valid``, failed rows from ``fill``."""
    if idx.size == n:
        return out_valid
    full = {}
    for key, a in out_valid.items():
        b = np.empty((n,) + a.shape[1:], dtype=a.dtype)
        b[...] = fill[key]
        b[idx] = a
        full[key] = b
    return full


# ---------------------------------------------------------------------------
# multi-device
# ---------------------------------------------------------------------------


def solve_sharded(batch: int, devices, solve_shard, out: dict) -> dict:
    """Contiguous shards of [0, batch) over ``devices``, one host thread each.

    ``solve_shard(slot, device, lo, hi, out_view)`` solves rows lo..hi into
    ``out_view`` (row views of ``out``). ``slot`` counts earlier occurrences
    of the same device in ``devices``, so a device listed twice gets two
    independent plans (one plan is never driven by two threads). Exceptions
    propagate after every shard has finished."""
    devices = list(devices)
    if not devices:
        raise ValueError("devices must be non-empty")
    shards = []
    for s, dev in enumerate(devices):
        lo, hi = shard_range(batch, s, len(devices))
        if hi > lo:
            shards.append((devices[:s].count(dev), dev, lo, hi))
    if len(shards) == 1:
        s, dev, lo, hi = shards[0]
        solve_shard(s, dev, lo, hi, {k: v[lo:hi] for k, v in out.items()})
        return out
    with ThreadPoolExecutor(max_workers=len(shards)) as ex:
        futs = [ex.submit(solve_shard, s, dev, lo, hi, {k: v[lo:hi] for k, v in out.items()})
                for s, dev, lo, hi in shards]
        errs = [f.exception() for f in futs]
    for e in errs:
        if e is not None:
            raise e
    return out
