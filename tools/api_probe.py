"""Where the Python API path spends its time (batch_newton_solve at 65,536)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
import paper_2605_14103_b200 as pf  # noqa: E402
from paper_2605_14103_b200 import hostmem  # noqa: E402
from paper_2605_14103_b200.fixtures import load_transmission  # noqa: E402
from paper_2605_14103_b200.results import TransmissionScenarios  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
net = load_transmission('gb2224')
m = pf.build_transmission_model(net)
base = pf.transmission_base(net, m.part)
plan = m.plan()
pt, qt = plan.scenarios(base, 10010, 0, B, 0.2, device=0)
hp, hq = hostmem.empty(tuple(pt.shape)), hostmem.empty(tuple(qt.shape))
hp[...] = pt.cpu().numpy()
hq[...] = qt.cpu().numpy()
scen = TransmissionScenarios(hp, hq)
for k in range(4):
    t0 = time.perf_counter()
    out = plan.alloc_outputs(B)
    t1 = time.perf_counter()
    plan.solve(hp, hq, 1e-8, 20, out=out)
    t2 = time.perf_counter()
    r = pf.batch_newton_solve(m, scen)
    t3 = time.perf_counter()
    print(f"alloc {1e3*(t1-t0):.1f} ms, C-ABI solve {1e3*(t2-t1):.1f} ms, batch_newton_solve {1e3*(t3-t2):.1f} ms",
          flush=True)
    del out, r
