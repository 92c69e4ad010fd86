"""Parity at scale against the REAL reference (tools/make_golden_scale.py).

256 GBnetwork scenarios (seed 10010) and 512 EULV scenarios (seed 10011),
generated on the device (bitwise the reference generator) and solved through
the C-ABI: flags and iteration counts equal the reference's for every
scenario (GMRES totals too for the GPU GMRES step), state summaries within
the parity tolerance, full states of every 32nd scenario within 1e-8.
"""

import numpy as np
import pytest

import paper_2605_14103_b200 as pf
from paper_2605_14103_b200 import engine
from paper_2605_14103_b200.fixtures import load_distribution, load_transmission

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gb():
    net = load_transmission("gb2224")
    model = pf.build_transmission_model(net)
    return model, pf.transmission_base(net, model.part)


def _nr_check(g, out):
    np.testing.assert_array_equal(out["converged"].astype(bool), g["converged"])
    np.testing.assert_array_equal(out["iterations"], g["iterations"])
    th, vm = out["theta"], out["vmag"]
    n = th.shape[1]
    assert np.abs(th.sum(1) - g["theta_sum"]).max() <= 1e-8 * n
    assert np.abs(vm.sum(1) - g["vmag_sum"]).max() <= 1e-8 * n
    assert np.abs(vm.min(1) - g["vmag_min"]).max() <= 1e-8
    assert np.abs(vm.max(1) - g["vmag_max"]).max() <= 1e-8
    k = g["keep"]
    assert np.abs(th[k] - g["theta"]).max() <= 1e-8
    assert np.abs(vm[k] - g["vmag"]).max() <= 1e-8


def test_nr_256_reference_scenarios(gb, golden):
    g = golden("scale_nr_gb2224")
    model, base = gb
    plan = model.plan()
    p, q = plan.scenarios(base, int(g["seed"]), 0, int(g["count"]), 0.2)
    out = plan.solve(p, q, 1e-8, 20)
    _nr_check(g, out)
    assert (out["final_mismatch_inf"] <= 1e-8).all()


def test_nr_gmres_step_256_reference_scenarios(gb, golden):
    g = golden("scale_nr_gb2224")
    model, base = gb
    plan = model.plan()
    plan.set_fd(model.y.csr, model.part.theta_block, model.part.q_block, 1e-6)
    p, q = plan.scenarios(base, int(g["seed"]), 0, int(g["count"]), 0.2)
    out = plan.solve_gmres(p, q, 1e-8, 20)
    _nr_check(g, out)
    np.testing.assert_array_equal(out["gmres_steps"].sum(1), g["gmres_total"])


def test_zbus_512_reference_scenarios(golden):
    g = golden("scale_zb_eulv")
    model = pf.build_zbus_model(load_distribution("eulv"))
    base = pf.distribution_base(model)
    plan = engine.zbus_plan_for(model)
    sw, sd = plan.scenarios(base, int(g["seed"]), 0, int(g["count"]), 0.2)
    out = plan.solve(sw, sd, 1e-9, 100)
    np.testing.assert_array_equal(out["converged"].astype(bool), g["converged"])
    np.testing.assert_array_equal(out["iterations"], g["iterations"])
    va = np.abs(out["v"])
    assert np.abs(va.sum(1) - g["vabs_sum"]).max() <= 1e-8 * va.shape[1]
    assert np.abs(va.min(1) - g["vabs_min"]).max() <= 1e-8
    assert np.abs(out["v"][g["keep"]] - g["v"]).max() <= 1e-8
    assert (out["residual_inf"] <= 1e-6).all()
