"""Z-Bus network reduction on the device vs the host path.

reduce_zbus(device=0) factors Y_NN with cuSOLVER getrf and solves for the
load columns Z[:, l] and v0 (acpf_zbus_reduce); the host path is LAPACK
getrf/getrs exactly as the reference (distribution.py:431-517). Both factor
with partial pivoting, so they agree to rounding; solves on the device-reduced
model must meet the same parity bar against the reference's golden vectors.
"""

import numpy as np
import pytest
import scipy.sparse

import paper_2605_14103_b200 as pf
from paper_2605_14103_b200 import distribution as dm
from paper_2605_14103_b200 import engine
from paper_2605_14103_b200.fixtures import load_distribution

pytestmark = pytest.mark.gpu

ZB = {"ieee13": "ieee13", "ieee123": "ieee123", "eulv": "eulv"}


@pytest.mark.parametrize("name", list(ZB))
def test_device_reduction_matches_host(name):
    net = load_distribution(ZB[name])
    host = pf.build_zbus_model(net)
    dev = pf.build_zbus_model(net, device=0)
    np.testing.assert_array_equal(dev.load_cols, host.load_cols)
    # rounding-level agreement: cond(Y_NN) is ~2e5 (IEEE13) to ~8e5 (EULV), so
    # two partial-pivoting LUs may differ by ~cond * eps relative
    zs = np.abs(host.z_load).max()
    assert np.abs(dev.z_load - host.z_load).max() <= 1e-10 * zs
    assert np.abs(dev.v0 - host.v0).max() <= 1e-10 * np.abs(host.v0).max()


@pytest.mark.parametrize("name", list(ZB))
def test_device_reduced_model_meets_parity(name, golden):
    g = golden(f"zb_{name}")
    model = pf.build_zbus_model(load_distribution(ZB[name]), device=0)
    out = engine.zbus_solve_arrays(model, g["s_wye"], g["s_delta"], 1e-9, 100)
    np.testing.assert_array_equal(out["converged"].astype(bool), g["converged"])
    np.testing.assert_array_equal(out["iterations"], g["iterations"])
    kv = g["v"].shape[0]
    assert np.abs(out["v"][:kv] - g["v"]).max() <= 1e-8


def test_device_reduction_singular():
    # an isolated non-slack phase (zero row/column) is singular on both paths
    y = scipy.sparse.csr_matrix(np.array([[2.0 - 1j, -1.0 + 0.5j, 0.0],
                                          [-1.0 + 0.5j, 2.0 - 1j, 0.0],
                                          [0.0, 0.0, 0.0]], dtype=complex))
    for device in (None, 0):
        with pytest.raises(dm.SingularYbusError):
            dm.reduce_zbus(y, [0], [1.0 + 0j], device=device)
