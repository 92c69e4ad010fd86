"""Host logic of the batched API (CPU): per-scenario isolation, array-backed
scenario/result sequences, and the threaded multi-device shard/gather.

The reference isolates a poisoned scenario instead of failing the batch
(batch.py:237-239, tests/test_batch.py:179-194; distribution.py:714-727);
these tests drive the same contract through batched solvers. The threaded
shard path (results.solve_sharded) is exercised with fake plans that write
their rows the way the C-ABI does.
"""

import threading

import numpy as np
import pytest

import paper_2605_14103_b200 as pf
from paper_2605_14103_b200 import batch as bt
from paper_2605_14103_b200 import results as rs
from paper_2605_14103_b200.fixtures import load_distribution, load_transmission
from paper_2605_14103_b200.shard import shard_range


@pytest.fixture(scope="module")
def tx():
    net = load_transmission("case14")
    m = pf.build_transmission_model(net)
    return m, pf.transmission_base(net, m.part)


def test_make_scenarios_stacked_and_bitwise(tx):
    model, base = tx
    spec = pf.ScenarioSpec(count=12, seed=1010)
    sc = pf.make_scenarios(base, spec)
    assert isinstance(sc, rs.TransmissionScenarios) and len(sc) == 12
    mult = pf.generate_load_multipliers(spec, base.n_elements)
    for k in range(12):
        ref = pf.apply_multipliers(base, mult[k])
        np.testing.assert_array_equal(sc[k].p_spec, ref.p_spec)
        np.testing.assert_array_equal(sc[k].q_spec, ref.q_spec)
    assert sc[3] is sc[3]  # memoised: identity holds, as for a list
    assert [s is t for s, t in zip(sc, list(sc))] == [True] * 12


def test_stack_checked_isolates_malformed(tx):
    model, base = tx
    sc = list(pf.make_scenarios(base, pf.ScenarioSpec(count=5, seed=4)))
    bad = pf.TransmissionScenario(p_spec=sc[2].p_spec[:-1], q_spec=sc[2].q_spec)
    worse = pf.TransmissionScenario(p_spec="x", q_spec=sc[3].q_spec)
    sc[2], sc[4] = bad, worse
    (p, q), idx, errors = rs.stack_checked(sc, ("p_spec", "q_spec"), (model.part.n_theta, model.part.n_q),
                                           np.float64, rs.TransmissionScenarios)
    assert list(idx) == [0, 1, 3] and sorted(errors) == [2, 4]
    assert errors[2].startswith("ValueError: scenario.p_spec must be a numeric vector")
    np.testing.assert_array_equal(p[2], sc[3].p_spec)


class _FakePlan:
    """Writes rows like the C-ABI does: theta = row sum of p, vmag = slot id."""

    def __init__(self, tag):
        self.tag = tag
        self.threads = set()

    def solve(self, p, q, tol, mx, out):
        self.threads.add(threading.get_ident())
        out["theta"][:] = p.sum(1, keepdims=True)
        out["vmag"][:] = self.tag
        out["converged"][:] = 1
        out["iterations"][:] = np.arange(p.shape[0])
        return out


@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 1, 2], [3, 3, 1, 0]])
def test_solve_sharded_gathers_in_order(devices):
    b = 37
    p = np.random.default_rng(1).normal(size=(b, 5))
    out = {"theta": np.zeros((b, 3)), "vmag": np.zeros((b, 3)), "converged": np.zeros(b, np.uint8),
           "iterations": np.zeros(b, np.int32)}
    plans = {}

    def shard(slot, dev, lo, hi, view):
        plan = plans.setdefault((dev, slot), _FakePlan(10 * dev + slot))
        plan.solve(p[lo:hi], None, 1e-8, 20, out=view)

    rs.solve_sharded(b, devices, shard, out)
    np.testing.assert_array_equal(out["theta"][:, 0], p.sum(1))
    assert out["converged"].all()
    assert len(plans) == len(devices)  # one plan per list entry, repeated devices included
    tags = out["vmag"][:, 0]
    for s, d in enumerate(devices):
        lo, hi = shard_range(b, s, len(devices))
        assert (tags[lo:hi] == 10 * d + devices[:s].count(d)).all()
        np.testing.assert_array_equal(out["iterations"][lo:hi], np.arange(hi - lo))


def test_solve_sharded_propagates_errors():
    def shard(slot, dev, lo, hi, view):
        if dev == 1:
            raise RuntimeError("device 1 failed")

    with pytest.raises(RuntimeError, match="device 1 failed"):
        rs.solve_sharded(10, [0, 1], shard, {"x": np.zeros(10)})


class _ListSolver:
    """A batched solver returning plain lists and raising on a poisoned scenario."""

    def __init__(self, poison):
        self.poison = poison
        self.calls = 0

    def solve_batch(self, scenarios):
        self.calls += 1
        out = []
        for sc in scenarios:
            if sc is self.poison:
                raise RuntimeError("boom")
            out.append(pf.FixedPointResult(v=np.zeros(2), converged=True, iterations=3, final_delta=0.0,
                                           residual_inf=1e-12))
        return out


def test_run_batch_isolates_poisoned_scenario_batched():
    scen = [object() for _ in range(5)]
    solver = _ListSolver(scen[2])
    rep = pf.run_batch(solver, scen, warmup=True)
    assert rep.n_converged == 4
    assert not rep.records[2].converged and "boom" in rep.records[2].error
    assert rep.results[2] is None
    assert [r.index for r in rep.records] == list(range(5))


def test_run_batch_warmup_guarded():
    scen = [object() for _ in range(3)]
    rep = pf.run_batch(_ListSolver(scen[0]), scen)  # the warm-up scenario itself is poisoned
    assert rep.n_converged == 2 and "boom" in rep.records[0].error


def test_run_batch_array_results_records():
    n = 6
    out = {"theta": np.zeros((n, 2)), "vmag": np.ones((n, 2)), "converged": np.array([1, 1, 0, 1, 0, 1], np.uint8),
           "iterations": np.array([3, 3, 1, 4, 20, 3], np.int32),
           "final_mismatch_inf": np.array([1e-10, 2e-10, 5.0, 3e-10, 1e-3, 1e-10]),
           "status": np.array([0, 0, 3, 0, 1, 0], np.int32)}
    errors = {5: "ValueError: bad scenario"}

    class S:
        def solve_batch(self, scen):
            return rs.NewtonResults(out, errors)

    rep = pf.run_batch(S(), list(range(n)), warmup=False)
    assert [r.converged for r in rep.records] == [True, True, False, True, False, False]
    assert rep.records[2].error == "voltage magnitude iterate collapsed to <= 0 (diverging)"
    assert rep.records[4].error is None and rep.records[4].iterations == 20
    assert rep.records[5].error == "ValueError: bad scenario" and rep.results[5] is None
    assert rep.results[3].iterations == 4 and rep.results[3].state.vmag[0] == 1.0
    d = pf.report_to_dict(rep)
    assert d["aggregate"]["n_converged"] == 3


def test_zbus_results_failed_rows_match_reference_record():
    model = pf.build_zbus_model(load_distribution("ieee13"))
    out = {"v": np.zeros((2, model.n), complex), "converged": np.array([1, 0], np.uint8),
           "iterations": np.array([12, 0], np.int32), "final_delta": np.array([1e-10, np.inf]),
           "residual_inf": np.array([1e-13, np.inf]), "status": np.array([0, -1], np.int32),
           "floor_slot": np.array([-1, -1], np.int32)}
    out["v"][1] = np.nan
    r = rs.ZbusResults(model, out, {1: "ValueError: scenario.wye_s must be a numeric vector"})
    bad = r[1]
    # the reference's _safe_zbus record (distribution.py:714-727)
    assert not bad.converged and bad.iterations == 0 and np.isnan(bad.v).all()
    assert bad.final_delta == np.inf and bad.residual_inf == np.inf
    assert bad.diagnostic.startswith("ValueError")
    assert r[0].converged and r[0].diagnostic is None
