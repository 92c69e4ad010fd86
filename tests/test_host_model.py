"""Host loaders/model builders vs the reference (golden vectors), CPU only."""

import json

import numpy as np
import pytest

import paper_2605_14103_b200 as pf
from paper_2605_14103_b200.fixtures import load_distribution, load_transmission, read_fixture

TX = {"case14": "case14", "case118": "case118", "case1354": "case1354pegase", "gb2224": "gb2224"}
ZB = {"ieee13": "ieee13", "ieee123": "ieee123", "eulv": "eulv"}


@pytest.mark.parametrize("tag", list(TX))
def test_ybus_partition_flat_start_bitwise(tag, golden):
    g = golden(f"nr_{tag}")
    m = pf.build_transmission_model(load_transmission(TX[tag]))
    y = m.y.csr
    np.testing.assert_array_equal(y.indptr, g["y_indptr"])
    np.testing.assert_array_equal(y.indices, g["y_indices"])
    # bitwise, signed zeros included (a plain == would accept -0.0 for +0.0)
    np.testing.assert_array_equal(y.data.view(np.uint64), g["y_data"].view(np.uint64))
    np.testing.assert_array_equal(m.part.theta_block, g["theta_block"])
    np.testing.assert_array_equal(m.part.q_block, g["q_block"])
    st = pf.flat_start(m.net, m.part)
    np.testing.assert_array_equal(st.theta, g["theta0"])
    np.testing.assert_array_equal(st.vmag, g["vmag0"])


@pytest.mark.parametrize("tag", list(TX))
def test_transmission_scenarios_bitwise(tag, golden):
    g = golden(f"nr_{tag}")
    net = load_transmission(TX[tag])
    m = pf.build_transmission_model(net)
    base = pf.transmission_base(net, m.part)
    np.testing.assert_array_equal(base.load_elements, g["load_elements"])
    count = g["multipliers"].shape[0]
    spec = pf.ScenarioSpec(count=count, seed=int(g["seed"]))
    mult = pf.generate_load_multipliers(spec, base.n_elements)
    np.testing.assert_array_equal(mult, g["multipliers"])
    p, q = pf.make_scenario_arrays(base, spec)
    np.testing.assert_array_equal(p, g["p_spec"])
    np.testing.assert_array_equal(q, g["q_spec"])
    # object path is the same numbers
    sc = pf.make_scenarios(base, pf.ScenarioSpec(count=3, seed=int(g["seed"])))
    np.testing.assert_array_equal(sc[2].p_spec, g["p_spec"][2])
    # a shard of rows equals the same rows of the full table
    p2, _ = pf.make_scenario_arrays(base, spec, start=count - 2, count=2)
    np.testing.assert_array_equal(p2, g["p_spec"][-2:])


@pytest.mark.parametrize("name", list(ZB))
def test_zbus_model_bitwise(name, golden):
    g = golden(f"zb_{name}")
    net = load_distribution(ZB[name])
    y = pf.build_three_phase_ybus(net)
    np.testing.assert_array_equal(y.indptr, g["y_indptr"])
    np.testing.assert_array_equal(y.indices, g["y_indices"])
    np.testing.assert_array_equal(y.data.view(np.uint64), g["y_data"].view(np.uint64))
    m = pf.build_zbus_model(net)
    np.testing.assert_array_equal(m.v0, g["v0"])
    np.testing.assert_array_equal(m.non_slack, g["non_slack"])
    for k in ("wye_idx", "delta_p", "delta_q", "wye_s", "delta_s"):
        np.testing.assert_array_equal(getattr(m, k), g[k])
    base = pf.distribution_base(m)
    count = g["multipliers"].shape[0]
    spec = pf.ScenarioSpec(count=count, seed=int(g["seed"]), target="distribution")
    sw, sd = pf.make_scenario_arrays(base, spec)
    np.testing.assert_array_equal(sw, g["s_wye"])
    np.testing.assert_array_equal(sd, g["s_delta"])


def test_zbus_load_columns(golden):
    g = golden("zb_ieee13")
    m = pf.build_zbus_model(load_distribution("ieee13"))
    np.testing.assert_array_equal(m.load_cols, g["load_cols"])
    assert np.abs(m.z_load - g["z_load"]).max() <= 1e-12 * np.abs(g["z_load"]).max()


def test_host_certificates_on_reference_solution(golden):
    g = golden("zb_ieee13")
    m = pf.build_zbus_model(load_distribution("ieee13"))
    sc = pf.DistributionScenario(m.wye_s, m.delta_s)
    assert pf.fixed_point_residual(m, sc, g["base_v"]) <= 1e-6
    assert pf.kirchhoff_residual(m, sc, g["base_v"]) <= 1e-8


def test_reference_csv_reader_and_profile(golden):
    import tempfile, os
    g = golden("zb_ieee13")
    m = pf.build_zbus_model(load_distribution("ieee13"))
    with tempfile.TemporaryDirectory() as td:
        p = os.path.join(td, "ref.csv")
        open(p, "w").write(read_fixture("ieee13_reference.csv"))
        ids, mags, _ = pf.read_reference_voltages(p)
    pos = {k: i for i, k in enumerate(m.reduced_ids())}
    got = np.array([abs(g["base_v"][pos[i]]) for i in ids])
    assert np.abs(got - mags).max() < 1e-3


def test_matpower_errors():
    bad = "function mpc = x\nmpc.baseMVA = 100;\nmpc.bus = [\n 1 3 0 0 0 0 1 1 0;\n];\n"
    with pytest.raises(pf.CaseParseError, match="missing mpc.gen"):
        pf.parse_matpower_case(bad)
    with pytest.raises(pf.CaseParseError, match="missing mpc.baseMVA"):
        pf.parse_matpower_case("mpc.bus = [1 3 0 0 0 0 1 1 0];")
    with pytest.raises(pf.CaseParseError, match="line 3"):
        pf.parse_matpower_case("mpc.baseMVA = 100;\nmpc.bus = [\n 1 3 x 0 0 0 1 1 0;\n];")


def test_txnet_json_roundtrip():
    net = load_transmission("case118")
    back = pf.network_from_json(pf.network_to_json(net))
    assert back.buses == net.buses and back.branches == net.branches


def test_distribution_schema_errors():
    doc = json.loads(read_fixture("ieee13.json"))
    doc["schema"] = "nope"
    with pytest.raises(pf.SchemaError, match=r"\$\.schema"):
        pf.parse_distribution_json(json.dumps(doc))
    doc = json.loads(read_fixture("ieee13.json"))
    doc["loads"][0]["bus"] = doc["slack"]["bus"]
    with pytest.raises(pf.SchemaError, match="slack bus"):
        pf.parse_distribution_json(json.dumps(doc))
    net = load_distribution("ieee13")
    again = pf.parse_distribution_json(pf.distribution_to_json(net))
    assert again.buses == net.buses and again.loads == net.loads


def test_branch_admittances_reproduce_branch_flows():
    # the table acpf_nr_plan_set_branches uploads gives the same flows as the
    # host branch_flows (reference transmission.py:453-481) at a random state
    from paper_2605_14103_b200 import engine
    from paper_2605_14103_b200 import transmission as tm
    net = load_transmission("case118")
    rng = np.random.default_rng(7)
    n = len(net.buses)
    st = tm.PolarState(rng.normal(0, 0.1, n), 1.0 + rng.normal(0, 0.02, n))
    f, t, y4, gs = engine.branch_admittances(net)
    u = st.vmag * np.exp(1j * st.theta)
    sf = u[f] * np.conj(y4[:, 0] * u[f] + y4[:, 1] * u[t])
    s_t = u[t] * np.conj(y4[:, 2] * u[f] + y4[:, 3] * u[t])
    hf, ht = tm.branch_flows(net, st)
    live = np.array([bool(b.status) for b in net.branches])
    np.testing.assert_allclose(sf, hf[live], rtol=0, atol=1e-13)
    np.testing.assert_allclose(s_t, ht[live], rtol=0, atol=1e-13)
    assert gs.shape == (n,)
