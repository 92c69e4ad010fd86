"""GPU parity on the failure branches, against reference-run goldens
(tools/make_golden_failures.py -> tests/golden/fail_nr.npz, fail_zb.npz).

Every case goes through the C-ABI (libacpf.so) as one stacked batch per
(tolerance, iteration cap), so the failing scenarios share launches with
converging ones and are masked per scenario on the device.

NR `_newton_loop` (reference transmission.py:333-380): non-finite exit
(:350-352), max_newton exit with iterations = max_newton and the fnorm of the
last check (:358-359, :380), V <= 0 collapse at iterations 1..10 (:355-357),
a loose tolerance. Z-Bus `_zbus_loop` (distribution.py:653-687):
VoltageFloorError on wye / delta phase / delta line-to-line sites at sweep 1
and mid-iteration (previous iterate returned, residual inf; :583-606,
:662-672), max_iter exits, a loose tolerance, a mixed batch.
"""

import numpy as np
import pytest

import paper_2605_14103_b200 as pf
from paper_2605_14103_b200 import engine
from paper_2605_14103_b200 import transmission as tm
from paper_2605_14103_b200.fixtures import load_transmission
from paper_2605_14103_b200.transmission import results_from_arrays

pytestmark = pytest.mark.gpu

TX = {"case14": "case14", "case118": "case118", "case1354": "case1354pegase", "gb2224": "gb2224"}


def _split(g, prefix):
    return {k.split("__", 1)[1]: v for k, v in g.items() if k.startswith(prefix + "__")}


def _solve_nr(model, d):
    """Solve every row of a failure set, one batch per (tol, max_newton)."""
    n = d["tol"].size
    out = {}
    keys = sorted({(float(t), int(m)) for t, m in zip(d["tol"], d["max_newton"])})
    rows = [None] * n
    for tol, mx in keys:
        idx = np.flatnonzero((d["tol"] == tol) & (d["max_newton"] == mx) & ~d["has_start"])
        o = model.plan().solve(np.ascontiguousarray(d["p_spec"][idx]), np.ascontiguousarray(d["q_spec"][idx]),
                               tol, mx)
        res = results_from_arrays(o)
        for j, s in enumerate(idx):
            rows[s] = res[j]
    out["res"] = rows
    return out


@pytest.mark.parametrize("tag", list(TX))
def test_nr_failure_branches(tag, golden):
    d = _split(golden("fail_nr"), tag)
    model = pf.build_transmission_model(load_transmission(TX[tag]))
    res = _solve_nr(model, d)["res"]
    for s, r in enumerate(res):
        lab = str(d["label"][s])
        if d["has_start"][s]:
            continue  # warm starts: test_nr_warm_start
        assert r.converged == bool(d["converged"][s]), lab
        assert r.iterations == int(d["iterations"][s]), lab
        assert (r.diagnostic or "") == str(d["diagnostic"][s]), lab
        ref_f = float(d["fnorm"][s])
        if np.isfinite(ref_f):
            # fnorm of the last check; at a converged exit both are below tol
            if r.converged:
                assert r.final_mismatch_inf <= float(d["tol"][s]), lab
            elif lab.startswith(("max_newton", "tol")):
                # (a stalled heavy-load trajectory, e.g. case1354 x2 running to
                # max_newton without collapsing, compares flags, iterations and
                # diagnostics only: after 20 non-contracting steps the iterates
                # of the exact and the inexact step are no longer comparable)
                # an unconverged iterate: the reference's GMRES step is inexact
                # (relative tolerance 1e-8, sparse.py:219-338), the engine's LU
                # step exact, so ||F|| of iterate k differs at ~1e-6 relative
                assert r.final_mismatch_inf == pytest.approx(ref_f, rel=1e-4), lab
        else:
            assert np.isnan(r.final_mismatch_inf) == np.isnan(ref_f), lab
            assert np.isinf(r.final_mismatch_inf) == np.isinf(ref_f), lab
        if r.converged:
            assert np.abs(r.state.theta - d["theta"][s]).max() <= 1e-8, lab
            assert np.abs(r.state.vmag - d["vmag"][s]).max() <= 1e-8, lab
        elif lab.startswith("max_newton"):
            # an unconverged iterate after 1-2 steps: the exact LU step and the
            # reference's inexact GMRES step (relative residual 1e-8) differ by
            # up to ~1e-7 here; the reference's own step on the GPU (below,
            # step="gmres") reproduces it within 1e-8
            assert np.abs(r.state.theta - d["theta"][s]).max() <= 1e-6, lab
            assert np.abs(r.state.vmag - d["vmag"][s]).max() <= 1e-6, lab


@pytest.mark.parametrize("tag", list(TX))
def test_nr_max_newton_gmres_step(tag, golden):
    """max_newton exits with the reference's own Newton step (GMRES-FD on the
    GPU): the unconverged iterate, its fnorm and iteration count match."""
    d = _split(golden("fail_nr"), tag)
    model = pf.build_transmission_model(load_transmission(TX[tag]))
    for mx in (1, 2):
        idx = np.flatnonzero((d["max_newton"] == mx) & (d["tol"] == 1e-8))
        scen = [pf.TransmissionScenario(d["p_spec"][s], d["q_spec"][s]) for s in idx]
        res = tm.batch_newton_solve(model, scen, tm.NewtonOptions(step="gmres", max_newton=mx))
        for s, r in zip(idx, res):
            assert not r.converged and r.iterations == int(d["iterations"][s]) == mx
            assert r.final_mismatch_inf == pytest.approx(float(d["fnorm"][s]), rel=1e-6)
            assert np.abs(r.state.theta - d["theta"][s]).max() <= 1e-8
            assert np.abs(r.state.vmag - d["vmag"][s]).max() <= 1e-8


def _zb_sets(g):
    return sorted({k.split("__", 1)[0] for k in g})


@pytest.mark.parametrize("key", ["wye_sweep1", "wye_sweep5", "delta_phase", "delta_phase_mid", "delta_line",
                                 "mixed_floor", "max_iter5", "tol1e-6", "eulv_max_iter5", "ieee123_floor",
                                 "ieee123_max_iter3"])
def test_zbus_failure_branches(key, golden):
    g = golden("fail_zb")
    assert key in _zb_sets(g)
    d = _split(g, key)
    net = pf.parse_distribution_json(str(d["network"]))
    model = pf.build_zbus_model(net, voltage_floor=float(d["floor"]))
    tol, mx = float(d["tol"]), int(d["max_iter"])
    out = engine.zbus_solve_arrays(model, d["s_wye"], d["s_delta"], tol, mx)
    res = engine.zbus_results(model, out)
    for s, r in enumerate(res):
        assert r.converged == bool(d["converged"][s]), s
        assert r.iterations == int(d["iterations"][s]), s
        assert (r.diagnostic or "") == str(d["diagnostic"][s]), s
        assert np.abs(r.v - d["v"][s]).max() <= 1e-8, s
        rd, rr = float(d["final_delta"][s]), float(d["residual"][s])
        if np.isfinite(rd):
            assert r.final_delta == pytest.approx(rd, rel=1e-6, abs=1e-12), s
        else:
            assert r.final_delta == rd, s
        if np.isfinite(rr) and rr > 1e-9:
            assert r.residual_inf == pytest.approx(rr, rel=1e-5), s
        elif np.isfinite(rr):
            assert r.residual_inf <= 1e-6, s
        else:
            assert r.residual_inf == rr, s


@pytest.mark.parametrize("tag", list(TX))
def test_nr_warm_start(tag, golden):
    """newton_solve(..., start=PolarState) / flat_start=False (reference
    transmission.py:306-330) through acpf_nr_solve_start: host buffers via the
    Python API, device buffers via the plan; flags, iterations and states."""
    d = _split(golden("fail_nr"), tag)
    rows = np.flatnonzero(d["has_start"])
    model = pf.build_transmission_model(load_transmission(TX[tag]))
    scen = [pf.TransmissionScenario(d["p_spec"][s], d["q_spec"][s]) for s in rows]
    starts = [pf.PolarState(d["theta0"][s], d["vmag0"][s]) for s in rows]
    res = tm.batch_newton_solve(model, scen, tm.NewtonOptions(flat_start=False), starts=starts)
    for s, r in zip(rows, res):
        assert r.converged == bool(d["converged"][s]) and r.iterations == int(d["iterations"][s]), s
        assert np.abs(r.state.theta - d["theta"][s]).max() <= 1e-8
        assert np.abs(r.state.vmag - d["vmag"][s]).max() <= 1e-8
    one = pf.newton_solve(model, scen[0], start=starts[0])
    assert one.iterations == int(d["iterations"][rows[0]])
    torch = pytest.importorskip("torch")
    cuda = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    out = model.plan().solve(cuda(d["p_spec"][rows]), cuda(d["q_spec"][rows]), 1e-8, 20,
                             theta_start=cuda(d["theta0"][rows]), vmag_start=cuda(d["vmag0"][rows]))
    np.testing.assert_array_equal(out["iterations"].cpu().numpy(), d["iterations"][rows])
    assert np.abs(out["vmag"].cpu().numpy() - d["vmag"][rows]).max() <= 1e-8
    # the flat start after a warm one (graph caches keyed on the start mode)
    flat = model.plan().solve(np.ascontiguousarray(d["p_spec"][rows]), np.ascontiguousarray(d["q_spec"][rows]),
                              1e-8, 20)
    assert flat["converged"].all()
    with pytest.raises(ValueError):
        pf.newton_solve(model, scen[0], tm.NewtonOptions(flat_start=False))
