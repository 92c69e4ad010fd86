"""CPU checks of the stop-rule tie-band classifier (tests/tiebands.py) and of
the decision margins recorded in the scale goldens (tools/make_golden_scale.py):
the recorded per-sweep / per-step values must reproduce the reference's own
iteration counts under its stop rules (distribution.py:674-679,
transmission.py:353)."""

import numpy as np
import pytest

from tiebands import BAND, classify, margins


def test_classify_separates_ties_from_real_mismatches():
    tol = 1e-9
    dec = np.array([[5e-3, 1e-6, 1e-9 * (1 + 1e-5), 8e-10],   # ref stops at 4; sweep 3 is a near-tie
                    [5e-3, 1e-6, 2e-9, 5e-10],                  # ref stops at 4, sweep 3 far from tol
                    [5e-3, 1e-6, 5e-10, np.nan]])               # ref stops at 3
    ref = np.array([4, 4, 3])
    got = np.array([3, 3, 3])
    ties, real = classify(ref, got, dec, tol)
    assert ties.tolist() == [0] and real.tolist() == [1]
    assert margins(ref, dec, tol) < BAND


@pytest.mark.parametrize("name", ["eulv", "ieee123", "ieee13"])
def test_scale_golden_zbus_decisions_reproduce_iterations(name, golden):
    g = golden(f"scale_zb_{name}")
    d, its = g["sweep_delta"], g["iterations"]
    tol = 1e-9
    for s in range(its.size):
        k = int(its[s])
        assert d[s, k - 1] <= tol and (k == 1 or (d[s, :k - 1] > tol).all()), s
    np.testing.assert_allclose(d[np.arange(its.size), its - 1], g["final_delta"], rtol=0, atol=0)
    # the smallest margin of any stop decision to tol, reported in DESIGN.md
    assert margins(its, d, tol) > 0


@pytest.mark.parametrize("name", ["gb2224", "case1354", "case118"])
def test_scale_golden_nr_decisions_reproduce_iterations(name, golden):
    g = golden(f"scale_nr_{name}")
    f, its = g["step_fnorm"], g["iterations"]
    for s in range(its.size):
        k = int(its[s])
        assert f[s, k] <= 1e-8 and (f[s, :k] > 1e-8).all(), s
    np.testing.assert_array_equal(f[np.arange(its.size), its], g["fnorm"])
    assert margins(its, f, 1e-8, first=0) > 0.5  # NR decisions are never near tol
