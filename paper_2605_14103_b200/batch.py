"""Seeded scenario batches and the batch driver (reference ``batch.py``).

Input format side of the hot path: the same counter-based multipliers
(Philox4x64-10 keyed by (seed, scenario index), reference batch.py:45-60),
the same load scaling (reference :121-151) and the same ``run_batch`` /
``BatchReport`` contract (reference :280-344). ``run_batch`` additionally
accepts a *batched* solver (an object with ``solve_batch(scenarios)``, e.g.
:class:`.transmission.GpuNewtonSolver` / :class:`.distribution` GPU solves):
the whole batch then goes to the device in one call and per-scenario
``wall_time`` is the batch time divided evenly.

:func:`make_scenario_arrays` builds the same scenarios directly as stacked
arrays (bitwise equal to stacking :func:`make_scenarios`; it performs the
identical IEEE multiply/subtract per element), which is what the C-ABI
consumes.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import Any, Callable, Sequence

import numpy as np

from . import hostmem

from .distribution import DistributionScenario, ZBusModel
from .network import BusPartition, TransmissionNetwork


_TARGETS = ("transmission", "distribution")


@dataclass(frozen=True)
class ScenarioSpec:
    """Seeded batch description (reference :25-42).

    ``count`` scenarios, 64-bit ``seed``, multipliers uniform on
    ``[1 - spread, 1 + spread)``, ``target`` the model family.
    """

    count: int
    seed: int
    spread: float = 0.2
    target: str = "transmission"

    def __post_init__(self):
        problems = (
            (self.count < 1, "count must be >= 1"),
            (not 0 <= self.spread < 1, "spread must satisfy 0 <= spread < 1"),
            (self.target not in _TARGETS, f"unknown target {self.target!r}"),
            (self.seed < 0, "seed must be a non-negative 64-bit integer"),
        )
        for bad, why in problems:
            if bad:
                raise ValueError(why)


def _uniform_row(seed: int, index: int, n: int) -> np.ndarray:
    """First ``n`` doubles of numpy's Philox4x64-10 stream keyed by (seed, index)."""
    key = np.array([seed, index], dtype=np.uint64)
    return np.random.Generator(np.random.Philox(key=key)).random(n)


def generate_load_multipliers(spec: ScenarioSpec, n_elements: int,
                              start: int = 0, count: int | None = None) -> np.ndarray:
    """Rows ``start .. start+count`` of the (count, n_elements) multiplier table.

    Row i is ``(1 - spread) + 2 spread * U_i`` (reference batch.py:45-60); it
    depends only on (seed, i), so a shard can build just its own rows. The
    device generator (``csrc/scenario_kernel.cu``) reproduces these bitwise.
    """
    rows = spec.count - start if count is None else count
    offset, scale = 1.0 - spec.spread, 2.0 * spec.spread
    table = np.empty((rows, n_elements))
    for r in range(rows):
        table[r] = offset + scale * _uniform_row(spec.seed, start + r, n_elements)
    return table


@dataclass(frozen=True)
class TransmissionBase:
    p_load: np.ndarray
    q_load: np.ndarray
    p_gen: np.ndarray
    q_gen: np.ndarray
    part: BusPartition
    load_elements: np.ndarray

    @property
    def n_elements(self) -> int:
        return int(self.load_elements.size)


@dataclass(frozen=True)
class DistributionBase:
    wye_s: np.ndarray
    delta_s: np.ndarray
    load_kinds: tuple

    @property
    def n_elements(self) -> int:
        return len(self.load_kinds)


def transmission_base(net: TransmissionNetwork, part: BusPartition) -> TransmissionBase:
    """Split loads from generation; elements = buses with nonzero load (:97-110)."""
    get = lambda name: np.array([getattr(b, name) for b in net.buses])  # noqa: E731
    pl, ql = get("p_load"), get("q_load")
    return TransmissionBase(pl, ql, get("p_gen"), get("q_gen"), part,
                            np.flatnonzero((pl != 0.0) | (ql != 0.0)))


def distribution_base(model: ZBusModel) -> DistributionBase:
    return DistributionBase(model.wye_s.copy(), model.delta_s.copy(), model.load_kinds)


def apply_multipliers(base, multipliers):
    """One scenario from one multiplier row (reference :121-151)."""
    from .transmission import TransmissionScenario

    m = np.asarray(multipliers, dtype=np.float64)
    if m.shape != (base.n_elements,):
        raise ValueError(f"expected {base.n_elements} multipliers, got shape {m.shape}")
    if isinstance(base, TransmissionBase):
        p, q = base.p_load.copy(), base.q_load.copy()
        p[base.load_elements] *= m
        q[base.load_elements] *= m
        return TransmissionScenario(p_spec=(base.p_gen - p)[base.part.theta_block],
                                    q_spec=(base.q_gen - q)[base.part.q_block])
    kinds = np.array(base.load_kinds)
    return DistributionScenario(wye_s=base.wye_s * m[kinds == "wye"],
                                delta_s=base.delta_s * m[kinds == "delta"])


def make_scenarios(base, spec: ScenarioSpec):
    """Full seeded batch as scenario objects (reference :154-159).

    Returned as a sequence of scenario objects backed by the stacked arrays
    (results.TransmissionScenarios / DistributionScenarios; every item is
    bitwise ``apply_multipliers(base, m_i)``), which the GPU solvers consume
    without re-stacking."""
    from .results import DistributionScenarios, TransmissionScenarios
    a, b = make_scenario_arrays(base, spec)
    cls = TransmissionScenarios if isinstance(base, TransmissionBase) else DistributionScenarios
    return cls(a, b)


def make_scenario_arrays(base, spec: ScenarioSpec, start: int = 0,
                         count: int | None = None, multipliers: np.ndarray | None = None):
    """Stacked scenario inputs for rows ``start .. start+count`` of ``spec``.

    Transmission: ``(p_spec[B, n_theta], q_spec[B, n_q])``; distribution:
    ``(s_wye[B, n_wye], s_delta[B, n_delta])`` complex. Element-for-element
    the same float operations as :func:`apply_multipliers`.
    """
    m = (generate_load_multipliers(spec, base.n_elements, start, count)
         if multipliers is None else np.asarray(multipliers, dtype=np.float64))
    if isinstance(base, TransmissionBase):
        b = m.shape[0]
        p = np.broadcast_to(base.p_load, (b, base.p_load.size)).copy()
        q = np.broadcast_to(base.q_load, (b, base.q_load.size)).copy()
        p[:, base.load_elements] *= m
        q[:, base.load_elements] *= m
        p = base.p_gen[None, :] - p
        q = base.q_gen[None, :] - q
        # page-locked result tables (hostmem): the solves copy them at PCIe rate
        op = hostmem.empty((b, base.part.theta_block.size))
        oq = hostmem.empty((b, base.part.q_block.size))
        np.take(p, base.part.theta_block, axis=1, out=op)
        np.take(q, base.part.q_block, axis=1, out=oq)
        return op, oq
    kinds = np.array(base.load_kinds)
    ow = hostmem.empty((m.shape[0], int((kinds == "wye").sum())), np.complex128)
    od = hostmem.empty((m.shape[0], int((kinds == "delta").sum())), np.complex128)
    np.multiply(base.wye_s[None, :], m[:, kinds == "wye"], out=ow)
    np.multiply(base.delta_s[None, :], m[:, kinds == "delta"], out=od)
    return ow, od


# ---------------------------------------------------------------------------
# Batch driver
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class ScenarioRecord:
    index: int
    converged: bool
    iterations: int
    residual: float
    wall_time: float
    error: str | None = None


@dataclass(frozen=True)
class BatchReport:
    records: tuple
    n_converged: int
    total_wall_time: float
    throughput: float
    worker_count: int
    results: tuple = field(repr=False, default=())


def _residual_of(res) -> float:
    """Transmission results carry ``final_mismatch_inf``, distribution ``residual_inf``."""
    name = next((k for k in ("final_mismatch_inf", "residual_inf") if hasattr(res, k)), None)
    return float("nan") if name is None else float(getattr(res, name))


def _record(index: int, res, wall: float, err: str | None) -> ScenarioRecord:
    if res is None:
        return ScenarioRecord(index, False, 0, float("inf"), wall, err)
    return ScenarioRecord(index, bool(res.converged), int(res.iterations), _residual_of(res),
                          wall, getattr(res, "diagnostic", None))


def _failure(exc: BaseException) -> str:
    return f"{type(exc).__name__}: {exc}"


def _run_batched(solver, scenarios, warmup: bool):
    """One device call for the whole batch; per-scenario time = total / count.

    Isolation as the reference's ``_timed_solve`` (batch.py:230-252): the
    warm-up never aborts the run; scenarios the solver rejects come back as
    records with ``error`` set and result ``None``; if the batched call itself
    raises, every scenario is re-solved on its own so only the poisoned ones
    fail."""
    if warmup:
        try:
            solver.solve_batch(scenarios[:1])
        except Exception:
            pass
    t0 = time.perf_counter()
    try:
        results = solver.solve_batch(scenarios)
    except Exception:
        results = None
    if results is None:
        outcomes = []
        for k in range(len(scenarios)):
            try:
                one = solver.solve_batch(scenarios[k:k + 1])
                errs = getattr(one, "errors", {}) or {}
                r, err = (None, errs[0]) if 0 in errs else (one[0], None)
            except Exception as exc:
                r, err = None, _failure(exc)
            outcomes.append((r, err))
        total = time.perf_counter() - t0
        share = total / len(scenarios)
        return [(r, share, err) for r, err in outcomes], total
    total = time.perf_counter() - t0
    share = total / len(scenarios)
    errors = getattr(results, "errors", {}) or {}
    if hasattr(results, "converged") and callable(results.converged):
        return _BatchedOutcome(results, share, errors), total
    return [(None, share, errors[k]) if k in errors else (r, share, None)
            for k, r in enumerate(results)], total


class _BatchedOutcome:
    """Array-backed outcomes of a batched solve (results.NewtonResults /
    ZbusResults): records are built from the stacked arrays, result objects
    only on demand."""

    def __init__(self, results, share: float, errors: dict):
        self.results, self.share, self.errors = results, share, errors

    def records(self) -> tuple:
        conv = self.results.converged()
        its = self.results.iterations()
        resid = self.results.residuals()
        diag = self.results.diagnostics()
        out = []
        for k in range(conv.size):
            if k in self.errors:
                out.append(ScenarioRecord(k, False, 0, float("inf"), self.share, self.errors[k]))
            else:
                out.append(ScenarioRecord(k, bool(conv[k]), int(its[k]), float(resid[k]), self.share, diag[k]))
        return tuple(out)

    def result_objects(self) -> tuple:
        return tuple(None if k in self.errors else self.results[k] for k in range(len(self.results)))


def _run_serial(solver, scenarios: list, warmup: bool):
    """Reference-style per-scenario callable, errors isolated per scenario."""
    if warmup:
        try:
            solver(scenarios[0])
        except Exception:
            pass
    done = []
    t0 = time.perf_counter()
    for sc in scenarios:
        t_sc = time.perf_counter()
        try:
            res, err = solver(sc), None
        except Exception as exc:
            res, err = None, _failure(exc)
        done.append((res, time.perf_counter() - t_sc, err))
    return done, time.perf_counter() - t0


def _report(outcomes, total: float, worker_count: int, keep_results: bool) -> BatchReport:
    if isinstance(outcomes, _BatchedOutcome):
        records = outcomes.records()
        results = outcomes.result_objects() if keep_results else ()
    else:
        records = tuple(_record(k, res, wall, err) for k, (res, wall, err) in enumerate(outcomes))
        results = tuple(res for res, _, _ in outcomes) if keep_results else ()
    return BatchReport(
        records=records,
        n_converged=sum(rec.converged for rec in records),
        total_wall_time=total,
        throughput=len(records) / total if total > 0 else float("inf"),
        worker_count=worker_count,
        results=results,
    )


def report_from_results(results, wall: float, worker_count: int = 1) -> BatchReport:
    """Report for results solved together in ``wall`` seconds (even time split)."""
    results = list(results)
    share = wall / len(results)
    return _report([(r, share, getattr(r, "diagnostic", None)) for r in results], wall,
                   worker_count, True)


def run_batch(
    solver: Callable[[Any], Any] | Any,
    scenarios: Sequence[Any],
    worker_count: int = 1,
    warmup: bool = True,
    keep_results: bool = True,
) -> BatchReport:
    """Solve every scenario in order and aggregate (reference :280-344).

    ``solver`` is a per-scenario callable (the reference's contract) or a
    batched solver with ``solve_batch(list) -> list`` (the GPU engine).
    ``worker_count`` is recorded only; the device sets its own parallelism.
    The optional one-scenario warm-up is not timed, as in the reference.
    """
    if worker_count < 1:
        raise ValueError("worker_count must be >= 1")
    if not hasattr(scenarios, "arrays"):
        scenarios = list(scenarios)
    if len(scenarios) == 0:
        raise ValueError("empty scenario batch")
    run = _run_batched if hasattr(solver, "solve_batch") else _run_serial
    outcomes, total = run(solver, scenarios, warmup)
    return _report(outcomes, total, worker_count, keep_results)


_REPORT_SCHEMA = "acpflow-batch-report/1"
_CSV_COLUMNS = ("index", "converged", "iterations", "residual", "error", "wall_time")


def report_to_dict(report: BatchReport) -> dict:
    """``acpflow-batch-report/1`` document (reference :352-376)."""
    aggregate = {"count": len(report.records), "n_converged": report.n_converged,
                 "worker_count": report.worker_count,
                 "timing": {"total_wall_time": report.total_wall_time,
                            "throughput": report.throughput}}
    records = [{"index": rec.index, "converged": rec.converged, "iterations": rec.iterations,
                "residual": rec.residual, "error": rec.error,
                "timing": {"wall_time": rec.wall_time}} for rec in report.records]
    return {"schema": _REPORT_SCHEMA, "aggregate": aggregate, "records": records}


def _csv_cells(rec: ScenarioRecord) -> tuple:
    err = (rec.error or "").replace(",", ";").replace("\n", " ")
    return (str(rec.index), str(int(rec.converged)), str(rec.iterations), repr(rec.residual),
            err, repr(rec.wall_time))


def report_to_csv(report: BatchReport) -> str:
    """One CSV row per scenario index, timing last (reference :379-387)."""
    rows = [",".join(_CSV_COLUMNS)] + [",".join(_csv_cells(rec)) for rec in report.records]
    return "\n".join(rows) + "\n"
