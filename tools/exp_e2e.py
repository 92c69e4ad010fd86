"""Probe: NR end-to-end (pinned host buffers through the C-ABI) vs chunking.

    ACPF_NR_CHUNK=16384 python tools/exp_e2e.py [B]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
import paper_2605_14103_b200 as pf  # noqa: E402
from paper_2605_14103_b200.fixtures import load_transmission  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
net = load_transmission('gb2224')
m = pf.build_transmission_model(net)
base = pf.transmission_base(net, m.part)
plan = m.plan()
pt, qt = plan.scenarios(base, 10010, 0, B, 0.2, device=0)
hp = torch.empty(pt.shape, dtype=pt.dtype, pin_memory=True)
hq = torch.empty(qt.shape, dtype=qt.dtype, pin_memory=True)
hp.copy_(pt)
hq.copy_(qt)
hp, hq = hp.numpy(), hq.numpy()
out = {k: torch.from_numpy(v).pin_memory().numpy() for k, v in plan.alloc_outputs(B).items()}
plan.solve(hp, hq, 1e-8, 20, out=out)
best = 1e30
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan.solve(hp, hq, 1e-8, 20, out=out)
    best = min(best, time.perf_counter() - t0)
print(f"chunk={os.environ.get('ACPF_NR_CHUNK', 'default')} B={B}: e2e {best * 1e3:.1f} ms "
      f"{int(out['converged'].sum()) / best:.0f} flows/s, kernel {plan.last_timing()[0]:.1f} ms", flush=True)
