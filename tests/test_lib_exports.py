"""The C-ABI library loads and exports every symbol include/acpf.h declares.

CPU-only: no compute calls that need a device, except the host-only symbolic
analysis entry (acpf_nr_analyze).
"""

import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2605_14103_b200 as pf
from paper_2605_14103_b200 import engine, transmission as tx
from paper_2605_14103_b200.fixtures import load_transmission

HEADER = Path(__file__).resolve().parents[1] / "include" / "acpf.h"


def declared():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(acpf_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported():
    lib = engine.load_library()
    names = declared()
    assert len(names) >= 12
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(engine.EXPORTED)


def test_abi_version_and_errors():
    lib = engine.load_library()
    assert lib.acpf_abi_version() == 1
    assert lib.acpf_device_count() >= 0
    h = C.c_void_p()
    rc = lib.acpf_nr_plan_create(0, 0, None, None, None, None, 0, None, 0, None, None, None, None,
                                 C.byref(h))
    assert rc == -1
    assert b"invalid" in lib.acpf_last_error()
    assert lib.acpf_nr_plan_destroy(None) == 0
    assert lib.acpf_zbus_plan_destroy(None) == 0


@pytest.mark.parametrize("case,expect,minfill", [("gb2224", 24273, (23165, 109233)),
                                                  ("case118", 807, (807, 1551))])
def test_symbolic_analysis_host_only(case, expect, minfill):
    m = pf.build_transmission_model(load_transmission(case), ordering="mmd")
    perm = tx.jacobian_ordering(m)
    info = engine.nr_analyze(m.y.csr, m.part.theta_block, m.part.q_block, perm)
    # 2x2-block factor over the non-slack buses; MMD: the SURVEY-pinned size
    assert info["n_j"] == m.part.n_theta
    assert info["nnz_lu"] == expect
    # the default (native minimum fill): no more fill, fewer block updates
    mf = pf.build_transmission_model(load_transmission(case))
    pmf = tx.jacobian_ordering(mf)
    assert sorted(pmf.tolist()) == list(range(m.part.n_theta))
    imf = engine.nr_analyze(mf.y.csr, mf.part.theta_block, mf.part.q_block, pmf)
    assert (imf["nnz_lu"], imf["n_pairs"]) == minfill
    assert imf["n_pairs"] <= info["n_pairs"] * 1.01
    built_in = engine.nr_analyze(m.y.csr, m.part.theta_block, m.part.q_block, None)
    assert built_in["nnz_lu"] == imf["nnz_lu"]
    md = engine.nr_ordering(m.y.csr, m.part.theta_block, engine.ORDER_MIN_DEGREE)
    assert engine.nr_analyze(m.y.csr, m.part.theta_block, m.part.q_block, md)["nnz_lu"] < 1.05 * expect
    with pytest.raises(engine.EngineError):
        engine.nr_ordering(m.y.csr, m.part.theta_block, 7)
    with pytest.raises(engine.EngineError):
        engine.nr_analyze(m.y.csr, m.part.theta_block, m.part.q_block, np.zeros_like(perm))


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    m = pf.build_transmission_model(load_transmission("case14"))
    with pytest.raises(engine.EngineUnavailable):
        pf.newton_solve(m)


@pytest.mark.parametrize("case", ["case14", "case118", "gb2224"])
def test_flat_start_lu_solves_dense_jacobian(case):
    """The LU shared by every scenario's first Newton step (host-built, what the
    device's step 0 substitutes with) solves the flat-start Jacobian of
    dense_jacobian (transmission.py:383-407) to rounding."""
    model = pf.build_transmission_model(load_transmission(case))
    st = tx.flat_start(model.net, model.part)
    j = tx.dense_jacobian(st, model.y, model.part)
    rhs = np.random.default_rng(7).standard_normal(j.shape[0])
    x = engine.nr_flat_start_solve(model.y.csr, model.part.theta_block, model.part.q_block, st.theta,
                                   st.vmag, rhs, perm=tx.jacobian_ordering(model))
    ref = np.linalg.solve(j, rhs)
    assert np.abs(x - ref).max() <= 1e-9 * max(1.0, np.abs(ref).max())
    assert np.abs(j @ x - rhs).max() <= 1e-9 * max(1.0, np.abs(rhs).max())
