"""Native report emission vs the reference's serialisers (CPU).

acpf_solve_result_json / acpf_report_csv (csrc/report.cpp) must write the
same bytes as json.dumps(doc, indent=1) of the reference's `solve`
document (cli.py:141-180 with report_to_dict, batch.py:352-376) and as
report_to_csv (batch.py:379-387): float repr, NaN/Infinity, signed zeros,
null rows, ensure_ascii escapes, the indent=1 layout.
"""

import json

import numpy as np
import pytest

from paper_2605_14103_b200 import batch as bm
from paper_2605_14103_b200 import engine


def _inputs(n=40, ns=6, seed=3):
    rng = np.random.default_rng(seed)
    conv = rng.random(n) < 0.7
    its = rng.integers(0, 21, n)
    res = rng.standard_normal(n) * 10.0 ** rng.integers(-20, 20, n)
    res[:10] = [np.nan, np.inf, -np.inf, 0.0, -0.0, 1e16, 1e-5, 1e15, 1e-4, 123456789012345678.0]
    errs = [None] * n
    errs[2] = 'V <= 0 at "bus 7"\n\tñ€\U0001F600,\x01\x7f'
    errs[11] = "maximum Newton iterations reached"
    a, b = rng.standard_normal((n, ns)), rng.standard_normal((n, ns))
    has = np.ones(n, bool)
    has[2] = False
    return conv, its, res, errs, a, b, has


def _reference_doc(kind, conv, its, res, errs, a, b, has, wall, ids=None):
    n = conv.size
    recs = [bm.ScenarioRecord(i, bool(conv[i]), int(its[i]), float(res[i]), wall / n, errs[i]) for i in range(n)]
    report = bm.BatchReport(records=tuple(recs), n_converged=int(conv.sum()), total_wall_time=wall,
                            throughput=n / wall, worker_count=1)
    if kind == "tx":
        sols = [{"index": i, "theta": list(a[i]) if has[i] else None, "vmag": list(b[i]) if has[i] else None}
                for i in range(n)]
    else:
        sols = {"node_phase_ids": ids,
                "records": [{"index": i, "v_re": list(a[i]) if has[i] else None,
                             "v_im": list(b[i]) if has[i] else None} for i in range(n)]}
    doc = {"schema": "acpflow-solve-result/1", "case": "x.m", "kind": kind, "seed": 9, "spread": 0.2,
           "batch": n, "report": bm.report_to_dict(report), "solutions": sols}
    return json.dumps(doc, indent=1) + "\n", bm.report_to_csv(report)


@pytest.mark.parametrize("kind", ["tx", "dist"])
def test_solve_result_json_bytes(kind, tmp_path):
    conv, its, res, errs, a, b, has = _inputs()
    ids = ["650.1", "632.2", "ñ.3"] if kind == "dist" else None
    wall = 0.0371
    ref_json, ref_csv = _reference_doc(kind, conv, its, res, errs, a, b, has, wall, ids)
    meta = {"case": "x.m", "kind": kind, "seed": 9, "spread": 0.2, "batch": conv.size,
            "total_wall_time": wall, "throughput": conv.size / wall}
    got = engine.solve_result_json(meta, conv, its, res, wall / conv.size, errs, a, b, has, ids)
    assert got == ref_json
    p = tmp_path / "r.json"
    assert engine.solve_result_json(meta, conv, its, res, wall / conv.size, errs, a, b, has, ids, path=p) is None
    assert p.read_text(encoding="utf-8") == ref_json
    assert engine.report_csv(conv, its, res, wall / conv.size, errs) == ref_csv


def test_float_repr_stress():
    rng = np.random.default_rng(11)
    x = np.concatenate([rng.standard_normal(50000) * 10.0 ** rng.integers(-300, 300, 50000),
                        rng.integers(-2 ** 53, 2 ** 53, 2000).astype(float), 10.0 ** np.arange(-30, 30),
                        [5e-324, 2.2250738585072014e-308, 1.7976931348623157e308, 0.1, 0.3, 2 / 3]])
    text = engine.report_csv(np.zeros(x.size, bool), np.zeros(x.size, int), x, 0.5)
    got = [line.split(",")[3] for line in text.splitlines()[1:]]
    assert got == [repr(float(v)) for v in x]


def test_empty_and_errors():
    meta = {"case": "x.m", "kind": "tx", "seed": 0, "spread": 0.0, "batch": 0, "total_wall_time": 0.0,
            "throughput": float("inf")}
    empty = engine.solve_result_json(meta, np.zeros(0, bool), np.zeros(0, int), np.zeros(0), 0.0)
    assert json.loads(empty)["solutions"] == [] and empty.endswith("]\n}\n")
    with pytest.raises(engine.EngineError):
        engine.solve_result_json(meta, np.ones(1, bool), np.ones(1, int), np.ones(1), 0.0, path="/nonexistent/x/y")
