"""Transmission Newton-Raphson: reference-shaped API over the GPU engine.

Mirrors reference ``pkg/src/acpflow/transmission.py``: ``PolarState``,
``TransmissionScenario``, ``NewtonOptions``, ``NewtonResult``,
``TransmissionModel``, ``flat_start``, ``base_scenario``, ``newton_solve``,
plus the batched entry ``batch_newton_solve`` the reference lacks (its batch
driver calls ``newton_solve`` per scenario).

The solve itself runs on the device (csrc/nr_kernel.cu): mismatch, Jacobian
assembly, static-pivot sparse LU refactorisation and triangular solves, the
whole Newton loop in one launch per scenario chunk. The step is an exact LU
solve instead of the reference's FD-preconditioned GMRES; the Newton
iterates agree with the reference to ~1e-12 and the flags/iteration counts
are identical (pinned by tests/golden).

Host-side helpers that the reference exposes publicly (``calc_injections``,
``mismatch``, ``dense_jacobian``, ``branch_flows``) are provided for
certificates and tests; they are not on the solve path.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .network import (AdmittanceMatrix, BusKind, BusPartition, TransmissionNetwork,
                      build_ybus, partition_buses)

_STATUS_TEXT = {
    2: "mismatch became non-finite (diverged iterate)",  # transmission.py:351
    3: "voltage magnitude iterate collapsed to <= 0 (diverging)",  # :356
}


@dataclass(frozen=True)
class PolarState:
    theta: np.ndarray
    vmag: np.ndarray

    def pack(self, part: BusPartition) -> np.ndarray:
        return np.concatenate([self.theta[part.theta_block], self.vmag[part.q_block]])

    def with_packed(self, x: np.ndarray, part: BusPartition) -> "PolarState":
        th, vm = self.theta.copy(), self.vmag.copy()
        th[part.theta_block] = x[: part.n_theta]
        vm[part.q_block] = x[part.n_theta:]
        return PolarState(th, vm)


@dataclass(frozen=True)
class TransmissionScenario:
    p_spec: np.ndarray
    q_spec: np.ndarray


@dataclass
class GmresOptions:
    """Accepted for API compatibility (reference sparse.py:186-200); unused:
    the engine's step solve is an exact LU."""

    tol: float = 1e-8
    restart: int = 60
    max_outer: int = 10


@dataclass
class NewtonOptions:
    """Reference transmission.py:100-117 plus ``step``: "lu" (default) solves
    each Newton step with the engine's exact sparse LU; "gmres" runs the
    reference's own step on the GPU (matrix-free GMRES with ``precond`` "fd"
    or "none", ``gmres`` and ``epsilon`` as in the reference)."""

    tol_mismatch: float = 1e-8
    max_newton: int = 20
    epsilon: float = 1e-6
    gmres: GmresOptions = field(default_factory=GmresOptions)
    flat_start: bool = True
    precond: str = "fd"
    step: str = "lu"

    def __post_init__(self):
        if not self.tol_mismatch > 0:
            raise ValueError("tol_mismatch must be positive")
        if self.max_newton < 1:
            raise ValueError("max_newton must be >= 1")
        if self.precond not in ("fd", "none"):
            raise ValueError(f"unknown preconditioner {self.precond!r}")
        if self.step not in ("lu", "gmres"):
            raise ValueError(f"unknown step solver {self.step!r}")


@dataclass(frozen=True)
class NewtonResult:
    state: PolarState
    converged: bool
    iterations: int
    final_mismatch_inf: float
    per_iteration_gmres: tuple = ()
    diagnostic: str | None = None

    @property
    def total_gmres_iterations(self) -> int:
        return sum(self.per_iteration_gmres)


@dataclass
class TransmissionModel:
    """Per-network artefacts (reference :134-160) plus the lazily built device plans."""

    net: TransmissionNetwork
    y: AdmittanceMatrix
    part: BusPartition
    ordering: str = "minfill"
    _plans: dict = field(default_factory=dict, repr=False)

    def plan(self, device: int = 0, slot: int = 0):
        """The device plan (one per (device, slot); a plan is driven by one
        host thread at a time, include/acpf.h)."""
        from . import engine
        key = device if slot == 0 else (device, slot)
        p = self._plans.get(key)
        if p is None:
            st = flat_start(self.net, self.part)
            perm = self._plans.get("_perm")
            if perm is None:
                perm = self._plans["_perm"] = jacobian_ordering(self)
            p = engine.NrPlan(self.y.csr, self.part.theta_block, self.part.q_block, st.theta,
                              st.vmag, device=device, perm=perm)
            self._plans[key] = p
        return p


def build_transmission_model(net: TransmissionNetwork, epsilon: float = 1e-6,
                             ordering: str = "minfill") -> TransmissionModel:
    """Y-bus + partition (reference :146-160). ``ordering`` of the sparse LU:
    'minfill' (native minimum fill, the default: fewest block updates),
    'md' (native minimum degree) or 'mmd' (SuperLU's MMD on A^T+A, the
    structure SURVEY.md pins the roofline's nnz_LU to)."""
    if ordering not in ("minfill", "md", "mmd"):
        raise ValueError(f"unknown ordering {ordering!r}")
    return TransmissionModel(net=net, y=build_ybus(net), part=partition_buses(net),
                             ordering=ordering)


def _as_model(net_or_model) -> TransmissionModel:
    if isinstance(net_or_model, TransmissionModel):
        return net_or_model
    return build_transmission_model(net_or_model)


def flat_start(net: TransmissionNetwork, part: BusPartition) -> PolarState:
    """Reference :169-177."""
    th = np.full(net.n, net.buses[part.slack[0]].theta_set)
    vm = np.ones(net.n)
    for k, b in enumerate(net.buses):
        if b.kind in (BusKind.SLACK, BusKind.PV):
            vm[k] = b.v_set
    return PolarState(th, vm)


def base_scenario(net: TransmissionNetwork, part: BusPartition) -> TransmissionScenario:
    """Reference :180-186."""
    p = np.array([b.p_inj for b in net.buses])
    q = np.array([b.q_inj for b in net.buses])
    return TransmissionScenario(p[part.theta_block], q[part.q_block])


def bus_pattern(model: TransmissionModel):
    """Pattern of the 2x2-block Jacobian: the Ybus pattern over the non-slack
    buses (theta-block order) plus the diagonal."""
    import scipy.sparse as sp
    tb = model.part.theta_block
    y = model.y.csr[tb][:, tb].tocsc()
    j = (abs(y) > 0).astype(np.float64) + sp.identity(tb.size, format="csc")
    j.data[:] = 1.0
    return j.tocsc()


def jacobian_ordering(model: TransmissionModel) -> np.ndarray:
    """Fill-reducing ordering of the non-slack bus graph (host, once).

    The engine factors the Jacobian as a matrix of 2x2 bus blocks
    [theta_i, V_i], so the ordering is computed on buses: the native greedy
    minimum fill / minimum degree of libacpf (acpf_nr_ordering), or, for
    ``ordering='mmd'``, SuperLU's MMD(A^T + A) permutation (only the
    permutation is taken from SuperLU; the factorisation runs on the device).
    perm[k] = theta-block position of the bus eliminated k-th.
    """
    if model.ordering in ("minfill", "md"):
        from . import engine
        kind = engine.ORDER_MIN_FILL if model.ordering == "minfill" else engine.ORDER_MIN_DEGREE
        return engine.nr_ordering(model.y.csr, model.part.theta_block, kind)
    import scipy.sparse as sp
    import scipy.sparse.linalg as spl
    j = bus_pattern(model)
    j = j + j.shape[0] * 4.0 * sp.identity(j.shape[0], format="csc")
    lu = spl.splu(j.tocsc(), permc_spec="MMD_AT_PLUS_A", diag_pivot_thresh=0.0,
                  options={"SymmetricMode": True})
    order = np.empty_like(lu.perm_c)
    order[lu.perm_c] = np.arange(lu.perm_c.size)
    return order.astype(np.int32)


# ---------------------------------------------------------------------------
# Solves
# ---------------------------------------------------------------------------


def stack_transmission_scenarios(model: TransmissionModel, scenarios) -> tuple:
    """Scenarios -> contiguous (p_spec[B, n_theta], q_spec[B, n_q]); raises on a malformed one."""
    (p, q), _, errors = _stack(model, scenarios)
    if errors:
        raise ValueError(next(iter(errors.values())))
    return p, q


def _stack(model: TransmissionModel, scenarios):
    from .results import TransmissionScenarios, stack_checked
    return stack_checked(scenarios, ("p_spec", "q_spec"), (model.part.n_theta, model.part.n_q),
                         np.float64, TransmissionScenarios)


def _check_options(opts: NewtonOptions | None, start) -> NewtonOptions:
    """Reference newton_solve (transmission.py:319-324): a start state is used
    as given; without one, flat_start=False is an error."""
    opts = opts or NewtonOptions()
    if start is None and not opts.flat_start:
        raise ValueError("flat_start=False requires an explicit start state")
    if start is not None and opts.step == "gmres":
        raise NotImplementedError("the GPU GMRES ablation solves from the flat start only")
    return opts


def status_diagnostic(out: dict, k: int):
    """The reference's diagnostic text for row k of the engine outputs
    (transmission.py:351, :356, :366-376; zero pivot: the engine's own)."""
    st = int(out["status"][k])
    if st in _STATUS_TEXT:
        return _STATUS_TEXT[st]
    if st == 4:
        return f"zero pivot in the static-pivot LU at Newton iteration {int(out['iterations'][k])}"
    if "gmres_diag" in out:
        kind, kk = int(out["gmres_diag"][k]), int(out["gmres_diag_k"][k])
        if kind == 1:
            return f"GMRES breakdown at Newton iteration {kk}"
        if kind == 2:
            return (f"GMRES stagnated at Newton iteration {kk} "
                    f"(relres {float(out['gmres_diag_relres'][k]):.2e})")
    return None


def results_from_arrays(out: dict, index=None) -> list:
    """Per-scenario NewtonResult records from the stacked engine outputs
    (with the GMRES step's per-iteration counts and diagnostics when present,
    transmission.py:366-376)."""
    from .results import NewtonResults
    res = NewtonResults(out)
    rng = range(len(res)) if index is None else index
    return [res[k] for k in rng]


_FAILED_ROW = {"converged": 0, "iterations": 0, "final_mismatch_inf": np.inf, "status": -1,
               "theta": np.nan, "vmag": np.nan}


def batch_newton_solve(net_or_model, scenarios, opts: NewtonOptions | None = None,
                       device: int | None = None, devices=None, starts=None):
    """Solve a list of scenarios on the GPU; order preserved.

    Each record equals ``newton_solve(model, scenario, opts)`` of the
    reference (flags, iteration counts; state within 1e-8). Returns a
    sequence of ``NewtonResult`` backed by the stacked outputs
    (results.NewtonResults). ``devices=[...]`` shards the batch into
    contiguous ranges over several GPUs (one plan and host thread each);
    ``device`` picks a single GPU. A malformed scenario becomes a failed
    record (NaN state, diagnostic = the error) instead of failing the batch,
    as the reference's batch driver isolates it (batch.py:237-239).
    ``starts``: a PolarState per scenario (or one for all) to start from
    instead of the flat start (reference ``start=``, transmission.py:306-330).
    """
    from .results import NewtonResults, scatter_rows, solve_sharded
    model = _as_model(net_or_model)
    opts = _check_options(opts, starts)
    if len(scenarios) == 0:
        return NewtonResults({k: np.empty((0,) if k not in ("theta", "vmag") else (0, len(model.net.buses)))
                              for k in _FAILED_ROW})
    (p, q), idx, errors = _stack(model, scenarios)
    devs = list(devices) if devices is not None else [0 if device is None else device]
    gm = opts.step == "gmres"
    b = p.shape[0]
    out = model.plan(devs[0]).alloc_outputs(b)
    if gm:
        out["gmres_steps"] = np.zeros((b, opts.max_newton), dtype=np.int32)
        out["gmres_diag"] = np.zeros(b, dtype=np.int32)
        out["gmres_diag_k"] = np.zeros(b, dtype=np.int32)
        out["gmres_diag_relres"] = np.zeros(b)

    th0 = vm0 = None
    if starts is not None:
        from . import hostmem
        st_list = [starts] * len(scenarios) if isinstance(starts, PolarState) else list(starts)
        if len(st_list) != len(scenarios):
            raise ValueError("starts must be one PolarState or one per scenario")
        n = len(model.net.buses)
        th0, vm0 = hostmem.empty((b, n)), hostmem.empty((b, n))
        for j, k in enumerate(idx):
            th0[j] = np.asarray(st_list[k].theta, dtype=np.float64)
            vm0[j] = np.asarray(st_list[k].vmag, dtype=np.float64)

    def shard(slot, dev, lo, hi, view):
        plan = model.plan(dev, slot)
        if th0 is not None:
            plan.solve(p[lo:hi], q[lo:hi], opts.tol_mismatch, opts.max_newton, out=view,
                       theta_start=th0[lo:hi], vmag_start=vm0[lo:hi])
            return
        if gm:
            if getattr(plan, "_fd_eps", None) != opts.epsilon:
                plan.set_fd(model.y.csr, model.part.theta_block, model.part.q_block, opts.epsilon)
            plan.solve_gmres(p[lo:hi], q[lo:hi], opts.tol_mismatch, opts.max_newton, opts.precond,
                             opts.gmres.tol, opts.gmres.restart, opts.gmres.max_outer, out=view)
        else:
            plan.solve(p[lo:hi], q[lo:hi], opts.tol_mismatch, opts.max_newton, out=view)

    if b:
        solve_sharded(b, devs, shard, out)
    fill = dict(_FAILED_ROW, gmres_steps=0, gmres_diag=0, gmres_diag_k=0, gmres_diag_relres=0.0)
    return NewtonResults(scatter_rows(out, idx, len(scenarios), fill), errors)


def newton_solve(net_or_model, scenario: TransmissionScenario | None = None,
                 opts: NewtonOptions | None = None, start: PolarState | None = None) -> NewtonResult:
    """Reference :306-330 (flat start, or ``start``), computed on the GPU."""
    model = _as_model(net_or_model)
    opts = _check_options(opts, start)
    if scenario is None:
        scenario = base_scenario(model.net, model.part)
    r = batch_newton_solve(model, [scenario], opts, starts=None if start is None else [start])
    if r.errors:
        raise ValueError(r.errors[0].split(": ", 1)[-1])
    return r[0]


class GpuNewtonSolver:
    """Batched solver object for :func:`.batch.run_batch` (``devices``: shard
    the batch over several GPUs, results.solve_sharded)."""

    def __init__(self, model: TransmissionModel, opts: NewtonOptions | None = None, device: int = 0,
                 devices=None):
        self.model = model
        self.opts = opts or NewtonOptions()
        self.device = device
        self.devices = list(devices) if devices is not None else None

    def solve_batch(self, scenarios):
        return batch_newton_solve(self.model, scenarios, self.opts, self.device, devices=self.devices)

    def __call__(self, scenario):
        return self.solve_batch([scenario])[0]


# ---------------------------------------------------------------------------
# Host helpers (public reference API; certificates/tests, not the solve path)
# ---------------------------------------------------------------------------


def calc_injections(state: PolarState, y: AdmittanceMatrix) -> tuple:
    """P, Q at every bus (reference :194-199)."""
    u = state.vmag * np.exp(1j * state.theta)
    s = u * np.conj(y.csr @ u)
    return s.real, s.imag


def mismatch(state: PolarState, scenario: TransmissionScenario, y: AdmittanceMatrix,
             part: BusPartition) -> np.ndarray:
    """F = [P - p_spec over theta block; Q - q_spec over PQ] (reference :202-215)."""
    p, q = calc_injections(state, y)
    return np.concatenate([p[part.theta_block] - scenario.p_spec, q[part.q_block] - scenario.q_spec])


def dense_jacobian(state: PolarState, y: AdmittanceMatrix, part: BusPartition) -> np.ndarray:
    """Explicit polar Jacobian on the free blocks (reference :383-407 formulas)."""
    yd = y.to_dense()
    e = np.exp(1j * state.theta)
    u = state.vmag * e
    i = yd @ u
    dth = 1j * u[:, None] * np.conj(np.diag(i) - yd * u[None, :])
    dv = u[:, None] * np.conj(yd * e[None, :]) + np.conj(np.diag(i)) * np.diag(e)
    tb, qb = part.theta_block, part.q_block
    return np.block([[dth.real[np.ix_(tb, tb)], dv.real[np.ix_(tb, qb)]],
                     [dth.imag[np.ix_(qb, tb)], dv.imag[np.ix_(qb, qb)]]])


def branch_flows(net: TransmissionNetwork, state: PolarState) -> tuple:
    """Complex power into each in-service branch at both ends (reference :453-481)."""
    idx = net.bus_index()
    u = state.vmag * np.exp(1j * state.theta)
    nbr = len(net.branches)
    sf = np.zeros(nbr, dtype=complex)
    stt = np.zeros(nbr, dtype=complex)
    for k, br in enumerate(net.branches):
        if not br.status:
            continue
        ys = 1.0 / complex(br.r, br.x)
        half_b = 0.5j * br.b_ch
        ratio = br.tap * np.exp(1j * br.shift)
        f, t = idx[br.from_bus], idx[br.to_bus]
        i_f = (ys + half_b) / (br.tap * br.tap) * u[f] + (-ys / np.conj(ratio)) * u[t]
        i_t = (-ys / ratio) * u[f] + (ys + half_b) * u[t]
        sf[k] = u[f] * np.conj(i_f)
        stt[k] = u[t] * np.conj(i_t)
    return sf, stt
