"""GPU parity: the CUDA path vs the reference's golden vectors (tests/golden).

Bar (BASELINE.json north star): identical convergence flags and iteration
counts; |dVm| <= 1e-8 p.u. and |dtheta| <= 1e-8 rad (Z-Bus: |dv| <= 1e-8 on
the complex node-phase voltage); final mismatch/residual below the
reference tolerance. All calls go through the C-ABI (libacpf.so).
"""

import numpy as np
import pytest

import paper_2605_14103_b200 as pf
from paper_2605_14103_b200 import engine
from paper_2605_14103_b200.fixtures import load_distribution, load_transmission

pytestmark = pytest.mark.gpu

TOL_V = 1e-8
TOL_TH = 1e-8

TX = {"case14": "case14", "case118": "case118", "case1354": "case1354pegase", "gb2224": "gb2224"}
ZB = {"ieee13": "ieee13", "ieee123": "ieee123", "eulv": "eulv"}


@pytest.fixture(scope="module")
def tx_models():
    return {k: pf.build_transmission_model(load_transmission(v)) for k, v in TX.items()}


@pytest.fixture(scope="module")
def zb_models():
    return {k: pf.build_zbus_model(load_distribution(v)) for k, v in ZB.items()}


@pytest.mark.parametrize("tag", list(TX))
def test_nr_matches_reference(tag, tx_models, golden):
    g = golden(f"nr_{tag}")
    model = tx_models[tag]
    out = model.plan().solve(np.ascontiguousarray(g["p_spec"]), np.ascontiguousarray(g["q_spec"]),
                             1e-8, 20)
    np.testing.assert_array_equal(out["converged"].astype(bool), g["converged"])
    np.testing.assert_array_equal(out["iterations"], g["iterations"])
    assert (out["final_mismatch_inf"] <= 1e-8).all()
    if "theta" in g:
        assert np.abs(out["theta"] - g["theta"]).max() <= TOL_TH
        assert np.abs(out["vmag"] - g["vmag"]).max() <= TOL_V


@pytest.mark.parametrize("tag", list(TX))
def test_nr_base_and_infeasible(tag, tx_models, golden):
    g = golden(f"nr_{tag}")
    model = tx_models[tag]
    r = pf.newton_solve(model)
    assert r.converged and r.iterations == int(g["base_iterations"])
    assert np.abs(r.state.theta - g["base_theta"]).max() <= TOL_TH
    assert np.abs(r.state.vmag - g["base_vmag"]).max() <= TOL_V
    sc = pf.base_scenario(model.net, model.part)
    h = pf.newton_solve(model, pf.TransmissionScenario(50 * sc.p_spec, 50 * sc.q_spec))
    assert h.converged == bool(g["huge_converged"])
    assert h.iterations == int(g["huge_iterations"])
    assert (h.diagnostic or "") == str(g["huge_diagnostic"])


def test_nr_pinned_entries_bit_exact(tx_models):
    model = tx_models["case118"]
    r = pf.newton_solve(model)
    for i in model.part.slack:
        assert r.state.theta[i] == model.net.buses[i].theta_set
        assert r.state.vmag[i] == model.net.buses[i].v_set
    for i in model.part.pv:
        assert r.state.vmag[i] == model.net.buses[i].v_set


def test_nr_batch_position_independent(tx_models, golden):
    g = golden("nr_case118")
    model = tx_models["case118"]
    p, q = g["p_spec"], g["q_spec"]
    perm = np.random.default_rng(3).permutation(p.shape[0])
    a = model.plan().solve(np.ascontiguousarray(p), np.ascontiguousarray(q), 1e-8, 20)
    b = model.plan().solve(np.ascontiguousarray(p[perm]), np.ascontiguousarray(q[perm]), 1e-8, 20)
    np.testing.assert_array_equal(a["theta"][perm], b["theta"])
    np.testing.assert_array_equal(a["vmag"][perm], b["vmag"])


@pytest.mark.parametrize("tag", list(ZB))
def test_zbus_matches_reference(tag, zb_models, golden):
    g = golden(f"zb_{tag}")
    model = zb_models[tag]
    out = engine.zbus_solve_arrays(model, g["s_wye"], g["s_delta"], 1e-9, 100)
    np.testing.assert_array_equal(out["converged"].astype(bool), g["converged"])
    np.testing.assert_array_equal(out["iterations"], g["iterations"])
    kv = g["v"].shape[0]
    assert np.abs(out["v"][:kv] - g["v"]).max() <= TOL_V
    assert (out["final_delta"][g["converged"]] <= 1e-9).all()
    assert (out["residual_inf"] <= 1e-6).all()


def test_zbus_noload_and_heavy(zb_models, golden):
    g = golden("zb_ieee13")
    model = zb_models["ieee13"]
    r = pf.zbus_iterate(model, pf.DistributionScenario(np.zeros_like(model.wye_s),
                                                       np.zeros_like(model.delta_s)))
    assert r.converged and r.iterations == int(g["noload_iterations"]) == 1
    np.testing.assert_array_equal(r.v, model.v0)
    h = pf.zbus_iterate(model, pf.DistributionScenario(model.wye_s * 60.0, model.delta_s * 60.0))
    assert h.converged == bool(g["heavy_converged"])
    assert h.iterations == int(g["heavy_iterations"])
    assert (h.diagnostic or "") == str(g["heavy_diagnostic"])


def test_zbus_batch_position_independent(zb_models, golden):
    g = golden("zb_ieee13")
    model = zb_models["ieee13"]
    sw, sd = g["s_wye"][:300], g["s_delta"][:300]
    perm = np.random.default_rng(5).permutation(300)
    a = engine.zbus_solve_arrays(model, sw, sd, 1e-9, 100)
    b = engine.zbus_solve_arrays(model, sw[perm], sd[perm], 1e-9, 100)
    np.testing.assert_array_equal(a["v"][perm], b["v"])
    np.testing.assert_array_equal(a["iterations"][perm], b["iterations"])


def test_nr_large_batch_consistent(tx_models, golden):
    """A large batch (many groups per level launch, long pipelines) gives the
    reference iteration count everywhere and the same bits as a small batch."""
    g = golden("nr_gb2224")
    model = tx_models["gb2224"]
    base = pf.transmission_base(model.net, model.part)
    p, q = pf.make_scenario_arrays(base, pf.ScenarioSpec(count=2048, seed=10010))
    out = model.plan().solve(p, q, 1e-8, 20)
    assert out["converged"].all() and (out["iterations"] == 4).all()
    np.testing.assert_array_equal(p[:8], g["p_spec"])
    small = model.plan().solve(np.ascontiguousarray(p[:8]), np.ascontiguousarray(q[:8]), 1e-8, 20)
    np.testing.assert_array_equal(small["theta"], out["theta"][:8])
    np.testing.assert_array_equal(small["vmag"], out["vmag"][:8])
    assert np.abs(out["vmag"][:8] - g["vmag"]).max() <= TOL_V


def test_zbus_large_batch_consistent(zb_models, golden):
    g = golden("zb_eulv")
    model = zb_models["eulv"]
    base = pf.distribution_base(model)
    sw, sd = pf.make_scenario_arrays(base, pf.ScenarioSpec(count=4096, seed=10011,
                                                           target="distribution"))
    out = engine.zbus_solve_arrays(model, sw, sd, 1e-9, 100)
    np.testing.assert_array_equal(out["iterations"][:64], g["iterations"])
    assert out["converged"].all() and (out["residual_inf"] <= 1e-6).all()
    small = engine.zbus_solve_arrays(model, sw[:8], sd[:8], 1e-9, 100)
    np.testing.assert_array_equal(small["v"], out["v"][:8])


# ---------------------------------------------------------------------------
# device scenario generation: bitwise the reference generator
# ---------------------------------------------------------------------------


def test_philox_multipliers_bitwise(golden):
    g = golden("philox")
    k = 0
    while f"m{k}" in g:
        seed, count, n = (int(x) for x in g[f"spec{k}"])
        got = engine.philox_multipliers(seed, 0, count, n, float(g[f"spread{k}"]))
        np.testing.assert_array_equal(got, g[f"m{k}"])
        k += 1
    # a shard of rows equals the same rows of the host table
    host = pf.generate_load_multipliers(pf.ScenarioSpec(count=300, seed=77), 1625)
    dev = engine.philox_multipliers(77, 200, 100, 1625, 0.2)
    np.testing.assert_array_equal(dev, host[200:])


@pytest.mark.parametrize("tag", ["case118", "gb2224"])
def test_nr_device_scenarios_bitwise(tag, tx_models, golden):
    g = golden(f"nr_{tag}")
    model = tx_models[tag]
    base = pf.transmission_base(model.net, model.part)
    count = g["p_spec"].shape[0]
    p, q = model.plan().scenarios(base, int(g["seed"]), 0, count)
    np.testing.assert_array_equal(p, g["p_spec"])
    np.testing.assert_array_equal(q, g["q_spec"])


@pytest.mark.parametrize("tag", ["ieee13", "ieee123", "eulv"])
def test_zbus_device_scenarios_bitwise(tag, zb_models, golden):
    g = golden(f"zb_{tag}")
    model = zb_models[tag]
    base = pf.distribution_base(model)
    count = min(256, g["s_wye"].shape[0])
    sw, sd = engine.zbus_plan_for(model).scenarios(base, int(g["seed"]), 0, count)
    np.testing.assert_array_equal(sw, g["s_wye"][:count])
    np.testing.assert_array_equal(sd, g["s_delta"][:count])


# ---------------------------------------------------------------------------
# edge cases: empty, single, ragged batches; chunked and pipelined host paths
# ---------------------------------------------------------------------------


def test_nr_empty_and_ragged_batches(tx_models, golden):
    g = golden("nr_case118")
    model = tx_models["case118"]
    plan = model.plan()
    p, q = np.ascontiguousarray(g["p_spec"]), np.ascontiguousarray(g["q_spec"])
    full = plan.solve(p, q, 1e-8, 20)
    empty = plan.solve(np.zeros((0, p.shape[1])), np.zeros((0, q.shape[1])), 1e-8, 20)
    assert empty["theta"].shape == (0, model.net.n)
    for b in (1, 7, 9, 17, 65):  # not multiples of the 8-scenario group
        out = plan.solve(np.ascontiguousarray(p[:b]), np.ascontiguousarray(q[:b]), 1e-8, 20)
        np.testing.assert_array_equal(out["theta"], full["theta"][:b])
        np.testing.assert_array_equal(out["vmag"], full["vmag"][:b])
        np.testing.assert_array_equal(out["iterations"], g["iterations"][:b])


@pytest.mark.parametrize("pipeline,chunk", [("0", "136"), ("1", "136"), ("2", "136"), ("2", "232"), ("2", "1000")])
def test_nr_chunked_and_pipelined_paths_agree(tx_models, monkeypatch, pipeline, chunk):
    # ragged chunks (ACPF_NR_CHUNK) through the host paths (0 serial, 1 copy
    # stream, 2 two concurrent chunk lanes) and the device-pointer path give
    # the same bits as one chunk
    torch = pytest.importorskip("torch")
    model = pf.build_transmission_model(load_transmission("case118"))
    base = pf.transmission_base(model.net, model.part)
    p, q = pf.make_scenario_arrays(base, pf.ScenarioSpec(count=1000, seed=1010))
    ref = model.plan().solve(p, q, 1e-8, 20)
    monkeypatch.setenv("ACPF_NR_CHUNK", chunk)  # 136: 8 chunks; 232: 5 (odd, ragged); 1000: one
    monkeypatch.setenv("ACPF_NR_PIPELINE", pipeline)
    model2 = pf.build_transmission_model(load_transmission("case118"))
    chunked = model2.plan().solve(p, q, 1e-8, 20)
    np.testing.assert_array_equal(chunked["theta"], ref["theta"])
    np.testing.assert_array_equal(chunked["iterations"], ref["iterations"])
    dev = model2.plan().solve(torch.from_numpy(p).cuda(), torch.from_numpy(q).cuda(), 1e-8, 20)
    np.testing.assert_array_equal(dev["vmag"].cpu().numpy(), ref["vmag"])


def test_zbus_empty_and_ragged_batches(zb_models, golden):
    g = golden("zb_ieee13")
    model = zb_models["ieee13"]
    sw, sd = np.ascontiguousarray(g["s_wye"][:200]), np.ascontiguousarray(g["s_delta"][:200])
    full = engine.zbus_solve_arrays(model, sw, sd, 1e-9, 100)
    empty = engine.zbus_solve_arrays(model, sw[:0], sd[:0], 1e-9, 100)
    assert empty["v"].shape == (0, model.n)
    for b in (1, 31, 33, 63, 65, 129):  # around the 32/64-scenario tiles
        out = engine.zbus_solve_arrays(model, sw[:b], sd[:b], 1e-9, 100)
        np.testing.assert_array_equal(out["v"], full["v"][:b])
        np.testing.assert_array_equal(out["iterations"], g["iterations"][:b])


@pytest.mark.parametrize("tag", ["case118", "gb2224"])
def test_nr_shared_first_step_matches_per_scenario_factor(tag, tx_models, golden, monkeypatch):
    """Step 0 on the flat-start LU shared by every scenario (nr_flat_start_factor)
    against step 0 factored per scenario (ACPF_NR_SHARED0=0): the same flags and
    iterations, states equal to rounding."""
    g = golden(f"nr_{tag}")
    model = tx_models[tag]
    p, q = np.ascontiguousarray(g["p_spec"]), np.ascontiguousarray(g["q_spec"])
    a = model.plan().solve(p, q, 1e-8, 20)
    monkeypatch.setenv("ACPF_NR_SHARED0", "0")
    per = _fresh_plan(model)
    b = per.solve(p, q, 1e-8, 20)
    np.testing.assert_array_equal(a["iterations"], b["iterations"])
    np.testing.assert_array_equal(a["converged"], b["converged"])
    assert np.abs(a["theta"] - b["theta"]).max() <= 1e-12
    assert np.abs(a["vmag"] - b["vmag"]).max() <= 1e-12
    # one step: the shared-LU step equals the per-scenario-factor step
    a1 = model.plan().solve(p, q, 1e-8, 1)
    b1 = per.solve(p, q, 1e-8, 1)
    assert np.abs(a1["theta"] - b1["theta"]).max() <= 1e-12
    assert np.abs(a1["vmag"] - b1["vmag"]).max() <= 1e-12


def _fresh_plan(model):
    """A new plan (model.plan() caches one per device) with the model's ordering;
    ACPF_NR_SHARED0 is read when the plan is created."""
    from paper_2605_14103_b200.transmission import flat_start, jacobian_ordering
    st = flat_start(model.net, model.part)
    return engine.NrPlan(model.y.csr, model.part.theta_block, model.part.q_block, st.theta, st.vmag,
                         perm=jacobian_ordering(model))


@pytest.mark.parametrize("tag", ["case14", "case118", "gb2224"])
def test_nr_without_dense_tail_matches_reference(tag, golden, monkeypatch):
    """The all-sparse factorisation (ACPF_NR_TAIL=0: no dense tail, every
    level through nr_factor_kernel) gives the reference's flags and
    iterations and states within 1e-8, like the default dense-tail path (on
    case14 the default tail is the whole matrix)."""
    monkeypatch.setenv("ACPF_NR_TAIL", "0")
    g = golden(f"nr_{tag}")
    model = pf.build_transmission_model(load_transmission(TX[tag]))
    out = model.plan().solve(np.ascontiguousarray(g["p_spec"]), np.ascontiguousarray(g["q_spec"]), 1e-8, 20)
    np.testing.assert_array_equal(out["converged"].astype(bool), g["converged"])
    np.testing.assert_array_equal(out["iterations"], g["iterations"])
    if "theta" in g:
        assert np.abs(out["theta"] - g["theta"]).max() <= TOL_TH
        assert np.abs(out["vmag"] - g["vmag"]).max() <= TOL_V
    sc = pf.base_scenario(model.net, model.part)
    h = model.plan().solve(np.ascontiguousarray(50 * sc.p_spec[None]), np.ascontiguousarray(50 * sc.q_spec[None]),
                           1e-8, 20)
    assert int(h["iterations"][0]) == int(g["huge_iterations"])
