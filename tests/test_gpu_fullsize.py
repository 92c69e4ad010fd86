"""Parity at BASELINE.json's full sizes through size-independent properties.

The bench batches (GBnetwork NR x 65,536, configs[2]; EULV Z-Bus x 262,144,
configs[3]) are too large for the reference to solve here, so they are
checked the way the domain allows at any size:

* the leading 4,096 / 16,384 rows are the reference's own scale-golden scenarios (seed
  10010 / 10011, tools/make_golden_scale.py): flags equal the reference's,
  iteration counts equal up to reported stop-rule ties (tests/tiebands.py),
  states within the north-star tolerance;
* those rows are bitwise the ones a small batch of the same scenarios gives
  (results independent of batch size and position);
* every scenario carries its certificate: NR final ||F||inf <= 1e-8 recomputed
  on the device from the returned state (acpf_nr_certify, independent of the
  solver's own stop test) and the slack power balance within n_theta *
  ||F||inf (test_transmission.py:398-416); Z-Bus final_delta <= tol, fixed-point
  residual <= 1e-6 (test_acceptance.py:217-240) and the Kirchhoff residual of
  distribution.py:624-630 on a slice of the tail of the batch;
* slack/PV entries are bit-exact their set points (test_transmission.py:389-396).
"""

import numpy as np
import pytest

import paper_2605_14103_b200 as pf
from paper_2605_14103_b200 import engine
from paper_2605_14103_b200.fixtures import load_distribution, load_transmission

from tiebands import check_iterations

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

NR_BATCH = 65536
ZB_BATCH = 262144
TOL = 1e-8


def test_nr_gb2224_full_batch(golden):
    model = pf.build_transmission_model(load_transmission("gb2224"))
    base = pf.transmission_base(model.net, model.part)
    plan = model.plan()
    plan.set_branches(model.net)
    p, q = plan.scenarios(base, 10010, 0, NR_BATCH, 0.2, device="cuda:0")
    out = plan.solve(p, q, 1e-8, 20)
    conv = out["converged"].bool()
    its = out["iterations"]
    assert bool(conv.all()), int((~conv).sum())
    assert bool((its == 4).all()), torch.unique(its).tolist()
    assert bool((out["status"] == 0).all())
    assert float(out["final_mismatch_inf"].max()) <= TOL
    # certificates recomputed from the returned state, every scenario
    cert = plan.certify(out["theta"], out["vmag"], p, q)
    assert float(cert["mismatch_inf"].max()) <= TOL
    # the slack balance residual is the sum of the non-slack P mismatches
    # (the reference bounds it by 1e-8 after a 1e-10 solve); at tol 1e-8 the
    # bound is n_theta * ||F||inf
    nth = model.part.n_theta
    assert float(cert["slack_balance"].abs().max()) <= nth * float(cert["mismatch_inf"].max()) + 1e-12
    # slack / PV entries bit-exact
    th, vm = out["theta"], out["vmag"]
    for i in model.part.slack:
        assert bool((th[:, i] == model.net.buses[i].theta_set).all())
        assert bool((vm[:, i] == model.net.buses[i].v_set).all())
    pv = torch.as_tensor(np.asarray(model.part.pv, dtype=np.int64), device=vm.device)
    vset = torch.as_tensor([model.net.buses[i].v_set for i in model.part.pv], dtype=torch.float64,
                           device=vm.device)
    assert bool((vm.index_select(1, pv) == vset).all())
    del cert
    # the leading rows are the reference's scale-golden scenarios
    g = golden("scale_nr_gb2224")
    n = int(g["count"])
    assert int(g["seed"]) == 10010
    np.testing.assert_array_equal(out["converged"][:n].cpu().numpy().astype(bool), g["converged"])
    ties = check_iterations("NR gb2224 x65536 (leading rows)", g["iterations"], its[:n].cpu().numpy(),
                            g["step_fnorm"], 1e-8, first=0)
    k = np.setdiff1d(g["keep"], ties)
    sel = np.searchsorted(g["keep"], k)
    assert np.abs(th[:n].cpu().numpy()[k] - g["theta"][sel]).max() <= TOL
    assert np.abs(vm[:n].cpu().numpy()[k] - g["vmag"][sel]).max() <= TOL
    # ... and bitwise what a small batch of the same scenarios gives, also
    # for a slice from the end of the batch
    for a in (0, NR_BATCH - 96):
        small = plan.solve(p[a:a + 96].contiguous(), q[a:a + 96].contiguous(), 1e-8, 20)
        assert torch.equal(small["theta"], th[a:a + 96])
        assert torch.equal(small["vmag"], vm[a:a + 96])


def test_zbus_eulv_full_batch(golden):
    model = pf.build_zbus_model(load_distribution("eulv"))
    base = pf.distribution_base(model)
    plan = engine.zbus_plan_for(model)
    plan.set_network(model)
    sw, sd = plan.scenarios(base, 10011, 0, ZB_BATCH, 0.2, device="cuda:0")
    sd = sd.reshape(ZB_BATCH, -1).contiguous()
    out = plan.solve(sw, sd, 1e-9, 100)
    its = out["iterations"]
    assert bool(out["converged"].bool().all())
    assert bool((out["status"] == 0).all())
    assert set(torch.unique(its).tolist()) <= {10, 11, 12}
    assert float(out["final_delta"].max()) <= 1e-9
    assert float(out["residual_inf"].max()) <= 1e-6
    # Kirchhoff certificate on the tail of the batch
    a = ZB_BATCH - 2048
    kcl = plan.kirchhoff(out["v"][a:].contiguous(), sw[a:].contiguous(), sd[a:].contiguous())
    assert float(kcl.max()) <= TOL
    g = golden("scale_zb_eulv")
    n = int(g["count"])
    assert int(g["seed"]) == 10011
    np.testing.assert_array_equal(out["converged"][:n].cpu().numpy().astype(bool), g["converged"])
    ties = check_iterations("Z-Bus eulv x262144 (leading rows)", g["iterations"], its[:n].cpu().numpy(),
                            g["sweep_delta"], 1e-9, first=1)
    v = out["v"]
    k = np.setdiff1d(g["keep"], ties)
    assert np.abs(v[:n].cpu().numpy()[k] - g["v"][np.searchsorted(g["keep"], k)]).max() <= TOL
    for a in (0, ZB_BATCH - 128):
        small = plan.solve(sw[a:a + 128].contiguous(), sd[a:a + 128].contiguous(), 1e-9, 100)
        assert torch.equal(small["v"], v[a:a + 128])
        assert torch.equal(small["iterations"], its[a:a + 128])
