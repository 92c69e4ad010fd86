"""Pin the CPU oracle (oracle/) to the reference's failure-branch goldens
(tools/make_golden_failures.py): the same flags, iteration counts, diagnostics
and states as the real reference on every failure path the GPU tests replay
(tests/test_gpu_failures.py). Same algorithm as the reference, so the bar is
tight: states within 1e-10 wherever they are finite.
"""

import numpy as np
import pytest

import paper_2605_14103_b200 as pf
from oracle import nr as onr
from oracle import zbus as ozb
from paper_2605_14103_b200.engine import zbus_floor_message
from paper_2605_14103_b200.fixtures import load_transmission

TX = {"case14": "case14", "case118": "case118", "case1354": "case1354pegase", "gb2224": "gb2224"}


def _split(g, prefix):
    return {k.split("__", 1)[1]: v for k, v in g.items() if k.startswith(prefix + "__")}


@pytest.mark.parametrize("tag", list(TX))
def test_oracle_nr_failures(tag, golden):
    d = _split(golden("fail_nr"), tag)
    m = pf.build_transmission_model(load_transmission(TX[tag]))
    st = pf.flat_start(m.net, m.part)
    case = onr.NrCase(m.y.csr, m.part.theta_block, m.part.q_block, st.theta, st.vmag)
    rows = range(d["tol"].size) if tag not in ("gb2224", "case1354") else range(0, d["tol"].size, 3)
    for s in rows:
        lab = str(d["label"][s])
        cs = case
        if "has_start" in d and d["has_start"][s]:  # warm start (transmission.py:306-330)
            cs = onr.NrCase(m.y.csr, m.part.theta_block, m.part.q_block, d["theta0"][s], d["vmag0"][s])
        with np.errstate(all="ignore"):
            o = onr.newton(cs, d["p_spec"][s], d["q_spec"][s], tol=float(d["tol"][s]),
                           max_newton=int(d["max_newton"][s]))
        assert o.converged == bool(d["converged"][s]), lab
        assert o.iterations == int(d["iterations"][s]), lab
        assert (o.diagnostic or "") == str(d["diagnostic"][s]), lab
        np.testing.assert_equal(np.isnan(o.final_mismatch_inf), np.isnan(d["fnorm"][s]))
        if np.isfinite(d["fnorm"][s]) and lab.startswith(("max_newton", "tol", "warm")):
            assert o.final_mismatch_inf == pytest.approx(float(d["fnorm"][s]), rel=1e-8), lab
            assert np.abs(o.theta - d["theta"][s]).max() <= 1e-10, lab
            assert np.abs(o.vmag - d["vmag"][s]).max() <= 1e-10, lab


@pytest.mark.parametrize("key", ["wye_sweep1", "wye_sweep5", "delta_phase", "delta_phase_mid", "delta_line",
                                 "mixed_floor", "max_iter5", "tol1e-6", "ieee123_floor", "ieee123_max_iter3"])
def test_oracle_zbus_failures(key, golden):
    d = _split(golden("fail_zb"), key)
    model = pf.build_zbus_model(pf.parse_distribution_json(str(d["network"])), voltage_floor=float(d["floor"]))
    case = ozb.ZbCase(model.y_nn, model.v0, model.wye_idx, model.delta_p, model.delta_q, model.voltage_floor)
    for s in range(d["iterations"].size):
        o = ozb.zbus(case, d["s_wye"][s], d["s_delta"][s], tol=float(d["tol"]), max_iter=int(d["max_iter"]))
        assert o.converged == bool(d["converged"][s]), s
        assert o.iterations == int(d["iterations"][s]), s
        diag = zbus_floor_message(model, o.v, o.floor_slot) if o.floor_slot >= 0 else ""
        assert diag == str(d["diagnostic"][s]), s
        assert np.abs(o.v - d["v"][s]).max() <= 1e-10, s
        np.testing.assert_equal(np.isinf(o.residual_inf), np.isinf(d["residual"][s]))
