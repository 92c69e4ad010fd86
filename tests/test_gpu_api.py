"""The reference-shaped Python API on the GPU: multi-plan sharding, per-scenario
isolation with the real batched solvers, and array-backed results.

* ``batch_newton_solve(..., devices=[0, 0])`` / ``batch_zbus_solve(...,
  devices=[0, 0])`` drive two plans on the one device from two host threads
  (results.solve_sharded); the gathered outputs are bitwise those of one plan.
* A malformed scenario inside a batch becomes a failed record (reference
  batch.py:237-239, distribution.py:714-727); the rest are solved as usual.
"""

import numpy as np
import pytest

import paper_2605_14103_b200 as pf
from paper_2605_14103_b200.fixtures import load_distribution, load_transmission

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gb():
    net = load_transmission("gb2224")
    m = pf.build_transmission_model(net)
    return m, pf.transmission_base(net, m.part)


def test_nr_two_plans_threaded_gather_bitwise(gb):
    model, base = gb
    sc = pf.make_scenarios(base, pf.ScenarioSpec(count=600, seed=10010))
    one = pf.batch_newton_solve(model, sc)
    two = pf.batch_newton_solve(model, sc, devices=[0, 0])
    for k in ("theta", "vmag", "converged", "iterations", "final_mismatch_inf", "status"):
        np.testing.assert_array_equal(one.out[k], two.out[k])
    assert one.converged().all() and (one.iterations() == 4).all()


def test_zbus_two_plans_threaded_gather_bitwise():
    model = pf.build_zbus_model(load_distribution("eulv"))
    base = pf.distribution_base(model)
    sc = pf.make_scenarios(base, pf.ScenarioSpec(count=300, seed=10011, target="distribution"))
    one = pf.batch_zbus_solve(model, sc)
    two = pf.batch_zbus_solve(model, sc, devices=[0, 0])
    for k in ("v", "converged", "iterations", "final_delta", "residual_inf", "status"):
        np.testing.assert_array_equal(one.out[k], two.out[k])


def test_run_batch_gpu_solver_isolates_malformed(gb):
    model, base = gb
    sc = list(pf.make_scenarios(base, pf.ScenarioSpec(count=9, seed=10010)))
    sc[4] = pf.TransmissionScenario(p_spec=sc[4].p_spec[:10], q_spec=sc[4].q_spec)
    rep = pf.run_batch(pf.GpuNewtonSolver(model), sc)
    assert rep.n_converged == 8
    assert rep.records[4].error.startswith("ValueError: scenario.p_spec")
    assert rep.results[4] is None
    assert all(rep.records[k].iterations == 4 for k in range(9) if k != 4)
    ref = pf.batch_newton_solve(model, [s for k, s in enumerate(sc) if k != 4])
    got = [rep.results[k] for k in range(9) if k != 4]
    for a, b in zip(ref, got):
        np.testing.assert_array_equal(a.state.vmag, b.state.vmag)


def test_batch_zbus_solve_isolates_malformed():
    model = pf.build_zbus_model(load_distribution("ieee13"))
    base = pf.distribution_base(model)
    sc = list(pf.make_scenarios(base, pf.ScenarioSpec(count=6, seed=5050, target="distribution")))
    sc[1] = pf.DistributionScenario(wye_s=np.zeros(3, complex), delta_s=sc[1].delta_s)
    res = pf.batch_zbus_solve(model, sc)
    assert not res[1].converged and res[1].iterations == 0 and np.isnan(res[1].v).all()
    assert res[1].diagnostic.startswith("ValueError")
    assert all(res[k].converged for k in (0, 2, 3, 4, 5))
