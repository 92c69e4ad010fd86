"""Time the solve-result document: native writer vs the Python json.dumps path.

    python tools/report_probe.py [batch]   (gb2224 on cuda:0; writes under /tmp)
"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, '.')
import paper_2605_14103_b200 as pf  # noqa: E402
from paper_2605_14103_b200 import batch as bm, engine  # noqa: E402
from paper_2605_14103_b200.fixtures import load_transmission  # noqa: E402
from paper_2605_14103_b200.results import NewtonResults  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
net = load_transmission('gb2224')
m = pf.build_transmission_model(net)
plan = m.plan()
base = pf.transmission_base(net, m.part)
pt, qt = plan.scenarios(base, 1010, 0, B, 0.2, device=0)
out = {k: v.cpu().numpy() for k, v in plan.solve(pt, qt, 1e-8, 20).items()}
res = NewtonResults(out)
wall = 1.0
meta = {"case": "gb2224.m", "kind": "tx", "seed": 1010, "spread": 0.2, "batch": B, "total_wall_time": wall,
        "throughput": B / wall}
t0 = time.perf_counter()
engine.solve_result_json(meta, res.converged(), res.iterations(), res.residuals(), wall / B, res.diagnostics(),
                         out["theta"], out["vmag"], path="/tmp/native.json")
t1 = time.perf_counter()
report = bm.report_from_results(res, wall)
doc = {"schema": "acpflow-solve-result/1", "case": "gb2224.m", "kind": "tx", "seed": 1010, "spread": 0.2,
       "batch": B, "report": bm.report_to_dict(report),
       "solutions": [{"index": i, "theta": list(r.state.theta), "vmag": list(r.state.vmag)}
                     for i, r in enumerate(res)]}
with open("/tmp/python.json", "w") as fh:
    fh.write(json.dumps(doc, indent=1) + "\n")
t2 = time.perf_counter()
same = open("/tmp/native.json", "rb").read() == open("/tmp/python.json", "rb").read()
size = len(open("/tmp/native.json", "rb").read())
print(f"gb2224 x {B}: document {size / 1e6:.0f} MB; native {t1 - t0:.2f} s, python json.dumps {t2 - t1:.2f} s "
      f"({(t2 - t1) / (t1 - t0):.1f}x); identical bytes: {same}")
