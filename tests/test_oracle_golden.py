"""Pin the CPU oracle (oracle/) to the real reference's golden vectors.

tests/golden/*.npz were produced by tools/make_golden.py running the
unmodified reference (acpflow) in the build container. Bar: identical flags
and iteration counts, states within 1e-10 (same algorithm, same LAPACK).
"""

import numpy as np
import pytest

from oracle import nr as onr
from oracle import scenarios as osc
from oracle import zbus as ozb
import paper_2605_14103_b200 as pf
from paper_2605_14103_b200.fixtures import load_distribution, load_transmission

TX = {"case14": "case14", "case118": "case118", "case1354": "case1354pegase", "gb2224": "gb2224"}


def nr_case(tag):
    m = pf.build_transmission_model(load_transmission(TX[tag]))
    st = pf.flat_start(m.net, m.part)
    return m, onr.NrCase(m.y.csr, m.part.theta_block, m.part.q_block, st.theta, st.vmag)


def zb_case(name):
    m = pf.build_zbus_model(load_distribution(name))
    return m, ozb.ZbCase(m.y_nn, m.v0, m.wye_idx, m.delta_p, m.delta_q, m.voltage_floor)


def test_philox_multipliers(golden):
    g = golden("philox")
    k = 0
    while f"m{k}" in g:
        seed, count, n = (int(x) for x in g[f"spec{k}"])
        got = osc.multipliers(seed, count, n, float(g[f"spread{k}"]))
        np.testing.assert_array_equal(got, g[f"m{k}"])
        k += 1
    assert k >= 3


def test_philox_survey_vectors():
    # SURVEY.md 8(c) golden vectors captured from numpy's Philox
    u = np.random.Generator(np.random.Philox(key=np.array([1010, 0], dtype=np.uint64))).random(4)
    assert u[0].hex() == "0x1.7fbc5f1dd3cdep-1"
    np.testing.assert_array_equal(osc.multipliers(1010, 1, 4)[0],
                                  [1.0997936143459455, 0.843203732834596, 1.0369119806461378,
                                   0.8126365959421643])


@pytest.mark.parametrize("tag,count", [("case14", 64), ("case118", 64), ("case1354", 4), ("gb2224", 3)])
def test_nr_oracle_matches_reference(tag, count, golden):
    g = golden(f"nr_{tag}")
    _, case = nr_case(tag)
    for k in range(count):
        o = onr.newton(case, g["p_spec"][k], g["q_spec"][k])
        assert o.converged == bool(g["converged"][k])
        assert o.iterations == int(g["iterations"][k])
        assert o.final_mismatch_inf <= 1e-8
        if "theta" in g:
            assert np.abs(o.theta - g["theta"][k]).max() < 1e-10
            assert np.abs(o.vmag - g["vmag"][k]).max() < 1e-10


@pytest.mark.parametrize("tag", ["case14", "case118"])
def test_nr_exact_lu_step_agrees(tag, golden):
    g = golden(f"nr_{tag}")
    _, case = nr_case(tag)
    for k in range(16):
        o = onr.newton(case, g["p_spec"][k], g["q_spec"][k], step="lu")
        assert o.converged and o.iterations == int(g["iterations"][k])
        assert np.abs(o.theta - g["theta"][k]).max() < 1e-9
        assert np.abs(o.vmag - g["vmag"][k]).max() < 1e-9


@pytest.mark.parametrize("tag", ["case14", "case118"])
def test_nr_infeasible_semantics(tag, golden):
    g = golden(f"nr_{tag}")
    m, case = nr_case(tag)
    sc = pf.base_scenario(m.net, m.part)
    o = onr.newton(case, 50 * sc.p_spec, 50 * sc.q_spec)
    assert o.converged == bool(g["huge_converged"])
    assert o.iterations == int(g["huge_iterations"])
    assert (o.diagnostic or "") == str(g["huge_diagnostic"])


@pytest.mark.parametrize("tag", ["case14", "case118"])
def test_sparse_jacobian_matches_reference_dense(tag, golden):
    g = golden(f"nr_{tag}")
    _, case = nr_case(tag)
    j = onr.sparse_jacobian(case, g["jac_theta"], g["jac_vmag"]).toarray()
    scale = np.abs(g["jac_dense"]).max()
    assert np.abs(j - g["jac_dense"]).max() <= 1e-13 * scale


@pytest.mark.parametrize("name,count", [("ieee13", 512), ("ieee123", 64), ("eulv", 4)])
def test_zbus_oracle_matches_reference(name, count, golden):
    g = golden(f"zb_{name}")
    _, case = zb_case(name)
    kv = g["v"].shape[0]
    for k in range(count):
        o = ozb.zbus(case, g["s_wye"][k], g["s_delta"][k])
        assert o.converged == bool(g["converged"][k])
        assert o.iterations == int(g["iterations"][k])
        assert abs(o.final_delta - g["final_delta"][k]) <= 1e-12
        if k < kv:
            assert np.abs(o.v - g["v"][k]).max() < 1e-12


def test_zbus_oracle_edge_cases(golden):
    g = golden("zb_ieee13")
    m, case = zb_case("ieee13")
    o = ozb.zbus(case, np.zeros_like(m.wye_s), np.zeros_like(m.delta_s))
    assert o.converged and o.iterations == 1
    np.testing.assert_array_equal(o.v, m.v0)
    h = ozb.zbus(case, m.wye_s * 60.0, m.delta_s * 60.0)
    assert h.converged == bool(g["heavy_converged"])
    assert h.iterations == int(g["heavy_iterations"])
