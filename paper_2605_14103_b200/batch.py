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

from .distribution import DistributionScenario, ZBusModel
from .network import BusPartition, TransmissionNetwork


@dataclass(frozen=True)
class ScenarioSpec:
    """count, 64-bit seed, multiplier half-range, target (reference :25-42)."""

    count: int
    seed: int
    spread: float = 0.2
    target: str = "transmission"

    def __post_init__(self):
        if self.count < 1:
            raise ValueError("count must be >= 1")
        if not 0 <= self.spread < 1:
            raise ValueError("spread must satisfy 0 <= spread < 1")
        if self.target not in ("transmission", "distribution"):
            raise ValueError(f"unknown target {self.target!r}")
        if self.seed < 0:
            raise ValueError("seed must be a non-negative 64-bit integer")


def generate_load_multipliers(spec: ScenarioSpec, n_elements: int,
                              start: int = 0, count: int | None = None) -> np.ndarray:
    """Rows ``start .. start+count`` of the (count, n_elements) multiplier table.

    Row i = (1 - spread) + 2 spread * U, U the first ``n_elements`` doubles of
    ``Generator(Philox(key=[seed, i]))`` (reference batch.py:45-60). ``start``
    lets a shard build only its own rows; every row depends only on
    (seed, i).
    """
    count = spec.count - start if count is None else count
    out = np.empty((count, n_elements))
    lo = 1.0 - spec.spread
    width = 2.0 * spec.spread
    for r in range(count):
        gen = np.random.Generator(
            np.random.Philox(key=np.array([spec.seed, start + r], dtype=np.uint64)))
        out[r] = lo + width * gen.random(n_elements)
    return out


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


def make_scenarios(base, spec: ScenarioSpec) -> list:
    """Full seeded batch as scenario objects (reference :154-159)."""
    mult = generate_load_multipliers(spec, base.n_elements)
    return [apply_multipliers(base, mult[i]) for i in range(spec.count)]


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
        return (np.ascontiguousarray(p[:, base.part.theta_block]),
                np.ascontiguousarray(q[:, base.part.q_block]))
    kinds = np.array(base.load_kinds)
    return (np.ascontiguousarray(base.wye_s[None, :] * m[:, kinds == "wye"]),
            np.ascontiguousarray(base.delta_s[None, :] * m[:, kinds == "delta"]))


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


@dataclass(frozen=True)
class _SlimOutcome:
    converged: bool
    iterations: int
    residual_inf: float
    diagnostic: str | None


def _residual_of(res) -> float:
    for name in ("final_mismatch_inf", "residual_inf"):
        if hasattr(res, name):
            return float(getattr(res, name))
    return float("nan")


def _record(index: int, res, wall: float, err: str | None) -> ScenarioRecord:
    if res is None:
        return ScenarioRecord(index, False, 0, float("inf"), wall, err)
    return ScenarioRecord(index, bool(res.converged), int(res.iterations), _residual_of(res),
                          wall, getattr(res, "diagnostic", None))


def _slim(res):
    return _SlimOutcome(bool(res.converged), int(res.iterations), _residual_of(res),
                        getattr(res, "diagnostic", None))


def run_batch(
    solver: Callable[[Any], Any] | Any,
    scenarios: Sequence[Any],
    worker_count: int = 1,
    warmup: bool = True,
    keep_results: bool = True,
) -> BatchReport:
    """Solve every scenario, preserve order, aggregate (reference :280-344).

    ``solver`` is either the reference-style per-scenario callable or a
    batched solver exposing ``solve_batch(list) -> list``; the GPU engine is
    the latter. ``worker_count`` is recorded; the device decides its own
    parallelism. Warm-up (one scenario) is excluded from timing, as in the
    reference.
    """
    if worker_count < 1:
        raise ValueError("worker_count must be >= 1")
    scenarios = list(scenarios)
    if not scenarios:
        raise ValueError("empty scenario batch")
    batched = hasattr(solver, "solve_batch")
    if batched:
        if warmup:
            solver.solve_batch(scenarios[:1])
        t0 = time.perf_counter()
        try:
            results = list(solver.solve_batch(scenarios))
            errs = [None] * len(results)
        except Exception as exc:  # whole-batch failure: isolate per record
            results = [None] * len(scenarios)
            errs = [f"{type(exc).__name__}: {exc}"] * len(scenarios)
        total = time.perf_counter() - t0
        per = total / len(scenarios)
        outcomes = [(r, per, e) for r, e in zip(results, errs)]
    else:
        if warmup:
            try:
                solver(scenarios[0])
            except Exception:
                pass
        outcomes = []
        t0 = time.perf_counter()
        for sc in scenarios:
            s0 = time.perf_counter()
            try:
                res, err = solver(sc), None
            except Exception as exc:
                res, err = None, f"{type(exc).__name__}: {exc}"
            outcomes.append((res, time.perf_counter() - s0, err))
        total = time.perf_counter() - t0
    records = tuple(_record(i, r, w, e) for i, (r, w, e) in enumerate(outcomes))
    kept = tuple(r for r, _, _ in outcomes) if keep_results else ()
    return BatchReport(
        records=records,
        n_converged=sum(r.converged for r in records),
        total_wall_time=total,
        throughput=len(records) / total if total > 0 else float("inf"),
        worker_count=worker_count,
        results=kept,
    )


def report_to_dict(report: BatchReport) -> dict:
    """``acpflow-batch-report/1`` (reference :352-376)."""
    return {
        "schema": "acpflow-batch-report/1",
        "aggregate": {
            "count": len(report.records),
            "n_converged": report.n_converged,
            "worker_count": report.worker_count,
            "timing": {"total_wall_time": report.total_wall_time,
                       "throughput": report.throughput},
        },
        "records": [
            {"index": r.index, "converged": r.converged, "iterations": r.iterations,
             "residual": r.residual, "error": r.error, "timing": {"wall_time": r.wall_time}}
            for r in report.records
        ],
    }


def report_to_csv(report: BatchReport) -> str:
    """CSV by scenario index, timing last (reference :379-387)."""
    out = ["index,converged,iterations,residual,error,wall_time"]
    for r in report.records:
        err = (r.error or "").replace(",", ";").replace("\n", " ")
        out.append(f"{r.index},{int(r.converged)},{r.iterations},{r.residual!r},{err},{r.wall_time!r}")
    return "\n".join(out) + "\n"
