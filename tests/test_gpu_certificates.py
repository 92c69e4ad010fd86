"""On-device certificates vs the reference and the host.

Reference anchor: tests/golden/cert.npz (tools/make_golden_certs.py) holds
the real reference's mismatch, branch_flows, calc_injections and
kirchhoff_residual at fixed converged and perturbed states; the device
certificates are evaluated at exactly those states
(test_*_certificates_match_reference).

NR: acpf_nr_certify's ||F||inf, slack power balance and branch loss against
the host `mismatch` / `branch_flows` (reference transmission.py:202-215,
:453-481) at the GPU-returned states; the balance identity of
test_transmission.py:398-416 holds for every scenario of a tight solve.
Z-Bus: acpf_zbus_kirchhoff against the host `kirchhoff_residual`
(distribution.py:624-630) and the reference acceptance bound (<= 1e-8,
test_acceptance.py:217-240).
"""

import numpy as np
import pytest

import paper_2605_14103_b200 as pf
from paper_2605_14103_b200 import engine
from paper_2605_14103_b200 import transmission as tm
from paper_2605_14103_b200.fixtures import load_distribution, load_transmission

pytestmark = pytest.mark.gpu


def _split(g, prefix):
    return {k.split("__", 1)[1]: v for k, v in g.items() if k.startswith(prefix + "__")}


@pytest.mark.parametrize("name", ["case118", "gb2224"])
def test_nr_certificates_match_reference(name, golden):
    d = _split(golden("cert"), f"nr_{name}")
    model = pf.build_transmission_model(load_transmission(name))
    plan = model.plan()
    plan.set_branches(model.net)
    p, q = np.ascontiguousarray(d["p_spec"]), np.ascontiguousarray(d["q_spec"])
    cert = plan.certify(np.ascontiguousarray(d["theta"]), np.ascontiguousarray(d["vmag"]), p, q)
    # sums of O(|Y| |u|^2) terms in a different order: rounding-level agreement
    np.testing.assert_allclose(cert["mismatch_inf"], d["mismatch_inf"], rtol=1e-11, atol=1e-12)
    np.testing.assert_allclose(cert["branch_loss"], d["branch_loss"], rtol=1e-11, atol=1e-12)
    ref_balance = d["p_slack"] - ((d["branch_loss"] + d["shunt_loss"]) - p.sum(axis=1))
    np.testing.assert_allclose(cert["slack_balance"], ref_balance, rtol=0, atol=1e-9)


@pytest.mark.parametrize("name", ["ieee13", "ieee123", "eulv"])
def test_zbus_kirchhoff_matches_reference(name, golden):
    d = _split(golden("cert"), f"zb_{name}")
    model = pf.build_zbus_model(load_distribution(name))
    plan = engine.zbus_plan_for(model)
    plan.set_network(model)
    kcl = plan.kirchhoff(np.ascontiguousarray(d["v"]), np.ascontiguousarray(d["s_wye"]),
                         np.ascontiguousarray(d["s_delta"]))
    # converged states sit at rounding noise (~1e-11, sums of O(|Y| |v|)
    # terms in another order); the perturbed ones are O(1e-3..1e2)
    np.testing.assert_allclose(kcl, d["kirchhoff"], rtol=1e-10, atol=1e-10)
    assert (d["kirchhoff"][d["v"].shape[0] // 2:] > 1e-6).all()


@pytest.mark.parametrize("name", ["case118", "gb2224"])
def test_nr_certificates_match_host(name, golden):
    tag = {"case118": "nr_case118", "gb2224": "nr_gb2224"}[name]
    g = golden(tag)
    model = pf.build_transmission_model(load_transmission(name))
    plan = model.plan()
    plan.set_branches(model.net)
    p = np.ascontiguousarray(g["p_spec"][:16])
    q = np.ascontiguousarray(g["q_spec"][:16])
    out = plan.solve(p, q, 1e-10, 20)
    assert out["converged"].all()
    cert = plan.certify(out["theta"], out["vmag"], p, q)
    slack = model.part.slack
    for k in range(p.shape[0]):
        st = tm.PolarState(out["theta"][k], out["vmag"][k])
        f = tm.mismatch(st, pf.TransmissionScenario(p[k], q[k]), model.y, model.part)
        assert abs(cert["mismatch_inf"][k] - np.abs(f).max()) <= 1e-12
        sf, stt = tm.branch_flows(model.net, st)
        loss = (sf + stt).sum().real
        assert abs(cert["branch_loss"][k] - loss) <= 1e-10 * max(1.0, abs(loss))
        pc, _ = tm.calc_injections(st, model.y)
        shunt = sum(b.gs * st.vmag[i] ** 2 for i, b in enumerate(model.net.buses))
        host_bal = pc[slack].sum() - ((loss + shunt) - p[k].sum())
        assert abs(cert["slack_balance"][k] - host_bal) <= 1e-9
        assert abs(cert["slack_balance"][k]) <= 1e-8  # the reference's bound
    assert (cert["mismatch_inf"] <= 1e-10).all()


def test_nr_certify_device_buffers(golden):
    torch = pytest.importorskip("torch")
    g = golden("nr_case118")
    model = pf.build_transmission_model(load_transmission("case118"))
    plan = model.plan()
    plan.set_branches(model.net)
    p = torch.from_numpy(np.ascontiguousarray(g["p_spec"][:64])).cuda()
    q = torch.from_numpy(np.ascontiguousarray(g["q_spec"][:64])).cuda()
    out = plan.solve(p, q, 1e-10, 20)
    cert = plan.certify(out["theta"], out["vmag"], p, q)
    host = plan.certify(out["theta"].cpu().numpy(), out["vmag"].cpu().numpy(), p.cpu().numpy(),
                        q.cpu().numpy())
    for k in cert:
        np.testing.assert_array_equal(cert[k].cpu().numpy(), host[k])


@pytest.mark.parametrize("name", ["ieee13", "ieee123", "eulv"])
def test_zbus_kirchhoff_matches_host(name, golden):
    g = golden(f"zb_{name}")
    model = pf.build_zbus_model(load_distribution(name))
    plan = engine.zbus_plan_for(model)
    plan.set_network(model)
    sw = np.ascontiguousarray(g["s_wye"][:32])
    sd = np.ascontiguousarray(g["s_delta"][:32])
    out = plan.solve(sw, sd, 1e-9, 100)
    kcl = plan.kirchhoff(out["v"], sw, sd)
    for k in range(sw.shape[0]):
        host = pf.kirchhoff_residual(model, pf.DistributionScenario(sw[k], sd[k]), out["v"][k])
        # both are rounding-level sums of O(|Y| |v|) terms: agree to 1e-10
        assert abs(kcl[k] - host) <= 1e-10 + 1e-6 * host
    assert (kcl[out["converged"].astype(bool)] <= 1e-8).all()


def test_zbus_kirchhoff_floor_is_inf():
    model = pf.build_zbus_model(load_distribution("ieee13"))
    plan = engine.zbus_plan_for(model)
    plan.set_network(model)
    v = np.ascontiguousarray(np.tile(model.v0, (2, 1)))
    v[1, model.wye_idx[0]] = 0.0  # a wye load's voltage at the floor
    sw = np.ascontiguousarray(np.tile(model.wye_s, (2, 1)))
    sd = np.ascontiguousarray(np.tile(model.delta_s, (2, 1)))
    kcl = plan.kirchhoff(v, sw, sd)
    assert np.isfinite(kcl[0]) and np.isinf(kcl[1])
