"""The reference's own Newton step on the GPU (SURVEY 8(f) #4 ablation).

NewtonOptions(step="gmres") runs matrix-free J v inside left-preconditioned
restarted GMRES with the fast-decoupled preconditioner, per scenario, through
acpf_nr_solve_gmres. Against the reference's golden vectors it must give the
same convergence flags, Newton iteration counts and total GMRES iterations
(`gmres_total`, NewtonResult.total_gmres_iterations) and states within 1e-8.
"""

import numpy as np
import pytest

import paper_2605_14103_b200 as pf
from paper_2605_14103_b200 import transmission as tm
from paper_2605_14103_b200.fixtures import load_transmission

pytestmark = pytest.mark.gpu

TX = {"case14": "case14", "case118": "case118", "case1354": "case1354pegase", "gb2224": "gb2224"}
GM = tm.NewtonOptions(step="gmres")


@pytest.mark.parametrize("tag", list(TX))
def test_gmres_step_matches_reference(tag, golden):
    g = golden(f"nr_{tag}")
    model = pf.build_transmission_model(load_transmission(TX[tag]))
    scen = [pf.TransmissionScenario(g["p_spec"][k], g["q_spec"][k]) for k in range(g["p_spec"].shape[0])]
    res = tm.batch_newton_solve(model, scen, GM)
    np.testing.assert_array_equal([r.converged for r in res], g["converged"])
    np.testing.assert_array_equal([r.iterations for r in res], g["iterations"])
    np.testing.assert_array_equal([r.total_gmres_iterations for r in res], g["gmres_total"])
    if "theta" in g:
        th = np.array([r.state.theta for r in res])
        vm = np.array([r.state.vmag for r in res])
        assert np.abs(th - g["theta"]).max() <= 1e-8
        assert np.abs(vm - g["vmag"]).max() <= 1e-8


@pytest.mark.parametrize("tag", ["case14", "case118"])
def test_gmres_step_base_and_infeasible(tag, golden):
    g = golden(f"nr_{tag}")
    model = pf.build_transmission_model(load_transmission(TX[tag]))
    r = tm.newton_solve(model, opts=GM)
    assert r.converged and r.iterations == int(g["base_iterations"])
    assert np.abs(r.state.vmag - g["base_vmag"]).max() <= 1e-8
    sc = pf.base_scenario(model.net, model.part)
    h = tm.newton_solve(model, pf.TransmissionScenario(50 * sc.p_spec, 50 * sc.q_spec), GM)
    assert h.converged == bool(g["huge_converged"])
    assert h.iterations == int(g["huge_iterations"])
    assert (h.diagnostic or "").split(" (relres")[0] == str(g["huge_diagnostic"]).split(" (relres")[0]


def test_gmres_without_preconditioner_same_newton_iterates():
    model = pf.build_transmission_model(load_transmission("case14"))
    base = pf.transmission_base(model.net, model.part)
    p, q = pf.make_scenario_arrays(base, pf.ScenarioSpec(count=40, seed=1010))
    scen = [pf.TransmissionScenario(p[k], q[k]) for k in range(40)]
    lu = tm.batch_newton_solve(model, scen)
    none = tm.batch_newton_solve(model, scen, tm.NewtonOptions(step="gmres", precond="none"))
    fd = tm.batch_newton_solve(model, scen, GM)
    assert [r.iterations for r in none] == [r.iterations for r in lu] == [r.iterations for r in fd]
    # the FD preconditioner needs fewer inner iterations than none
    assert sum(r.total_gmres_iterations for r in fd) < sum(r.total_gmres_iterations for r in none)
