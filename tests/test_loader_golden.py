"""Host loaders vs the reference on 850 mutated inputs (CPU only).

tests/golden/loader_cases.json.gz holds mutated case14 MATPOWER texts and
IEEE13 feeder documents with the REAL reference's outcome for each
(tools/make_golden_parsers.py): the same error type and message, or the same
parsed buses/loads, a bitwise-equal Y-bus and v0 within 1e-12.
"""

import gzip
import hashlib
import json
import logging
from pathlib import Path

import numpy as np
import pytest

import paper_2605_14103_b200 as pf

CASES = json.loads(gzip.open(Path(__file__).parent / "golden" / "loader_cases.json.gz", "rt").read())


def _digest(y) -> str:
    y = y.tocsr()
    y.sort_indices()
    h = hashlib.sha256()
    for a in (y.indptr, y.indices, y.data):
        h.update(a.tobytes())
    return h.hexdigest()


def _matpower(text: str) -> dict:
    try:
        net = pf.parse_matpower_case(text)
        y = pf.build_ybus(net).complex_csr()
    except Exception as exc:  # noqa: BLE001
        return {"error": type(exc).__name__, "message": str(exc)}
    return {"name": net.name, "notes": list(net.notes), "ignored": list(net.ignored_fields),
            "buses": [[b.id, b.kind.value, b.v_set, b.p_gen, b.q_gen] for b in net.buses],
            "n_branches": len(net.branches), "ybus": _digest(y)}


def _feeder(text: str, expect: dict) -> None:
    try:
        net = pf.parse_distribution_json(text)
    except Exception as exc:  # noqa: BLE001
        assert {"error": type(exc).__name__, "message": str(exc)} == expect
        return
    assert "error" not in expect, expect
    assert [list(b) for b in net.buses] == expect["buses"]
    assert net.slack_bus == expect["slack"]
    assert [[ld.kind, ld.bus, ld.phases, ld.s.real, ld.s.imag] for ld in net.loads] == expect["loads"]
    try:
        y = pf.build_three_phase_ybus(net)
        assert _digest(y) == expect["ybus"]
        m = pf.build_zbus_model(net)
    except Exception as exc:  # noqa: BLE001
        assert (type(exc).__name__, str(exc)) == (expect["model_error"], expect["model_message"])
        return
    assert "model_error" not in expect, expect
    v0 = np.array([complex(*z) for z in expect["v0"]])
    assert np.abs(m.v0 - v0).max() <= 1e-12 * max(1.0, np.abs(v0).max())


@pytest.fixture(autouse=True)
def _quiet_demotions(caplog):
    caplog.set_level(logging.ERROR)


@pytest.mark.parametrize("k", [k for k, c in enumerate(CASES) if c["kind"] == "matpower"])
def test_matpower_case_matches_reference(k):
    assert _matpower(CASES[k]["text"]) == CASES[k]["expect"]


@pytest.mark.parametrize("k", [k for k, c in enumerate(CASES) if c["kind"] == "feeder"])
def test_feeder_document_matches_reference(k):
    _feeder(CASES[k]["text"], CASES[k]["expect"])


def test_cases_cover_both_outcomes():
    for kind in ("matpower", "feeder"):
        sub = [c["expect"] for c in CASES if c["kind"] == kind]
        assert sum("error" in e for e in sub) >= 50 and sum("error" not in e for e in sub) >= 20
    assert any("model_error" in c["expect"] for c in CASES)  # singular Y_NN after a dropped line
