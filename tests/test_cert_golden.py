"""Pin the host certificate restatements to the reference (CPU).

tests/golden/cert.npz (tools/make_golden_certs.py) holds what the real
reference computes at fixed states -- its own converged states and the same
states perturbed: ||mismatch||inf (transmission.py:202-215), the branch loss
(branch_flows, :453-481), the slack injection (calc_injections, :194-199),
the bus shunt loss, and kirchhoff_residual (distribution.py:624-630). The
package's host functions must reproduce them; the device certificates are
checked against the same numbers in tests/test_gpu_certificates.py.
"""

import numpy as np
import pytest

import paper_2605_14103_b200 as pf
from paper_2605_14103_b200 import transmission as tm
from paper_2605_14103_b200.fixtures import load_distribution, load_transmission


def _split(g, prefix):
    return {k.split("__", 1)[1]: v for k, v in g.items() if k.startswith(prefix + "__")}


@pytest.mark.parametrize("name", ["case118", "gb2224"])
def test_host_nr_certificates_match_reference(name, golden):
    d = _split(golden("cert"), f"nr_{name}")
    model = pf.build_transmission_model(load_transmission(name))
    slack = model.part.slack[0]
    for k in range(d["theta"].shape[0]):
        st = tm.PolarState(d["theta"][k], d["vmag"][k])
        f = tm.mismatch(st, pf.TransmissionScenario(d["p_spec"][k], d["q_spec"][k]), model.y, model.part)
        assert np.abs(f).max() == pytest.approx(d["mismatch_inf"][k], rel=1e-12, abs=1e-13)
        sf, stt = tm.branch_flows(model.net, st)
        assert (sf + stt).sum().real == pytest.approx(d["branch_loss"][k], rel=1e-12, abs=1e-13)
        pc, _ = tm.calc_injections(st, model.y)
        assert pc[slack] == pytest.approx(d["p_slack"][k], rel=1e-12, abs=1e-13)


@pytest.mark.parametrize("name", ["ieee13", "ieee123", "eulv"])
def test_host_kirchhoff_matches_reference(name, golden):
    d = _split(golden("cert"), f"zb_{name}")
    model = pf.build_zbus_model(load_distribution(name))
    for k in range(d["v"].shape[0]):
        host = pf.kirchhoff_residual(model, pf.DistributionScenario(d["s_wye"][k], d["s_delta"][k]), d["v"][k])
        assert host == pytest.approx(d["kirchhoff"][k], rel=1e-10, abs=1e-12)
