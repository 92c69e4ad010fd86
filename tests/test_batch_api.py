"""Batch driver contract (reference batch.py:280-387) on the host."""

import json

import numpy as np
import pytest

import paper_2605_14103_b200 as pf


class _Res:
    def __init__(self, k):
        self.converged = k % 3 != 0
        self.iterations = k % 5
        self.residual_inf = float(k)
        self.diagnostic = None if self.converged else "x"


class _Batched:
    def __init__(self):
        self.calls = []

    def solve_batch(self, scenarios):
        self.calls.append(len(scenarios))
        return [_Res(s) for s in scenarios]


def test_run_batch_per_scenario_callable():
    rep = pf.run_batch(lambda s: _Res(s), list(range(10)))
    assert [r.index for r in rep.records] == list(range(10))
    assert rep.n_converged == sum(1 for k in range(10) if k % 3)
    assert rep.records[3].error == "x" and rep.records[3].residual == 3.0


def test_run_batch_batched_solver_one_call():
    b = _Batched()
    rep = pf.run_batch(b, list(range(7)), keep_results=False)
    assert b.calls == [1, 7]  # warm-up then the whole batch in one call
    assert rep.results == ()
    assert [r.iterations for r in rep.records] == [k % 5 for k in range(7)]


def test_poisoned_scenario_isolated():
    def solver(s):
        if s == 2:
            raise ValueError("boom")
        return _Res(s)

    rep = pf.run_batch(solver, list(range(4)), warmup=False)
    assert rep.records[2].error == "ValueError: boom" and not rep.records[2].converged


def test_report_serialisation():
    rep = pf.run_batch(lambda s: _Res(s), list(range(3)), warmup=False)
    d = pf.report_to_dict(rep)
    assert d["schema"] == "acpflow-batch-report/1" and d["aggregate"]["count"] == 3
    json.dumps(d)
    csv = pf.report_to_csv(rep).splitlines()
    assert csv[0] == "index,converged,iterations,residual,error,wall_time" and len(csv) == 4


def test_spec_validation():
    with pytest.raises(ValueError):
        pf.ScenarioSpec(count=0, seed=1)
    with pytest.raises(ValueError):
        pf.ScenarioSpec(count=1, seed=1, spread=1.0)
    with pytest.raises(ValueError):
        pf.NewtonOptions(tol_mismatch=0)
    with pytest.raises(ValueError):
        pf.FixedPointOptions(max_iter=0)
