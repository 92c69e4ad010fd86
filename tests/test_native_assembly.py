"""Native model build vs the NumPy restatement (CPU).

acpf_ybus_build / acpf_y3_build (csrc/assemble.cpp) must give the same CSR,
bit for bit (indptr, indices, value bits incl. signed zeros), as
build_ybus_host / build_three_phase_ybus_host, which restate the
reference's network.py:450-496 and distribution.py:356-391. The reference
itself is checked on 850 mutated inputs by tests/test_loader_golden.py
(which now runs through the native builders).
"""

import gzip
import json
from pathlib import Path

import numpy as np
import pytest

import paper_2605_14103_b200 as pf
from paper_2605_14103_b200 import distribution as ds
from paper_2605_14103_b200 import engine
from paper_2605_14103_b200 import network as nw
from paper_2605_14103_b200.fixtures import load_distribution, load_transmission

CASES = json.loads(gzip.open(Path(__file__).parent / "golden" / "loader_cases.json.gz", "rt").read())


def _bits(y):
    y = y.tocsr()
    return y.indptr.astype(np.int64).tolist(), y.indices.tolist(), y.data.view(np.int64).tolist()


@pytest.mark.parametrize("name", ["case14", "case118", "case1354pegase", "gb2224"])
def test_ybus_native_bitwise(name):
    net = load_transmission(name)
    assert _bits(nw.build_ybus(net).csr) == _bits(nw.build_ybus_host(net).csr)


@pytest.mark.parametrize("name", ["ieee13", "ieee123", "eulv"])
def test_three_phase_native_bitwise(name):
    net = load_distribution(name)
    assert _bits(ds.build_three_phase_ybus(net)) == _bits(ds.build_three_phase_ybus_host(net))


def test_native_on_mutated_inputs():
    n_tx = n_d = 0
    for case in CASES:
        text = case.get("text") or case.get("input")
        if text is None:
            continue
        kind = case.get("kind", "")
        try:
            net = pf.parse_matpower_case(text) if "matpower" in kind or text.lstrip().startswith("function") \
                else pf.parse_distribution_json(text)
        except Exception:  # noqa: BLE001 - parser rejections are test_loader_golden's business
            continue
        if isinstance(net, pf.TransmissionNetwork):
            try:
                host = nw.build_ybus_host(net).csr
            except Exception as exc:  # noqa: BLE001
                with pytest.raises(type(exc)):
                    nw.build_ybus(net)
                continue
            assert _bits(nw.build_ybus(net).csr) == _bits(host)
            n_tx += 1
        else:
            assert _bits(ds.build_three_phase_ybus(net)) == _bits(ds.build_three_phase_ybus_host(net))
            n_d += 1
    assert n_tx + n_d > 100


def test_ybus_native_errors_and_edges():
    net = load_transmission("case14")
    br = net.branches[0]
    bad = pf.TransmissionNetwork(**{**net.__dict__, "branches": [type(br)(**{**br.__dict__, "r": 0.0, "x": 0.0})]
                                    + list(net.branches[1:])})
    with pytest.raises(pf.CaseParseError, match="has r = x = 0"):
        nw.build_ybus(bad)
    # a lone bus: no branches, no shunts -> an empty 1 x 1 CSR
    y = engine.ybus_build(1, [], [], [], [], [], [], [], [], [0.0], [0.0])
    assert y.shape == (1, 1) and y.nnz == 0
    assert engine.y3_build(3, []).nnz == 0
    with pytest.raises(engine.EngineError):
        engine.ybus_build(2, [0], [5], [0.1], [0.1], [0.0], [1.0], [0.0], [1], [0.0, 0.0], [0.0, 0.0])
