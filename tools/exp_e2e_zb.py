"""Probe: EULV Z-Bus end-to-end (pinned host buffers through the C-ABI) vs chunking.

    ACPF_ZBUS_CHUNK=16384 python tools/exp_e2e_zb.py [B]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
import paper_2605_14103_b200 as pf  # noqa: E402
from paper_2605_14103_b200 import engine  # noqa: E402
from paper_2605_14103_b200.fixtures import load_distribution  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
m = pf.build_zbus_model(load_distribution('eulv'))
base = pf.distribution_base(m)
plan = engine.zbus_plan_for(m)
sw, sd = plan.scenarios(base, 10011, 0, B, 0.2, device=0)
hsw = torch.empty(sw.shape, dtype=sw.dtype, pin_memory=True)
hsw.copy_(sw)
hsd = torch.empty((B, max(1, sd.shape[1])), dtype=sd.dtype, pin_memory=True)[:, :sd.shape[1]].contiguous()
hsw, hsd = hsw.numpy(), hsd.numpy()
out = {k: torch.from_numpy(v).pin_memory().numpy() for k, v in plan.alloc_outputs(B).items()}
plan.solve(hsw, hsd, 1e-9, 100, out=out)
best = 1e30
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan.solve(hsw, hsd, 1e-9, 100, out=out)
    best = min(best, time.perf_counter() - t0)
print(f"chunk={os.environ.get('ACPF_ZBUS_CHUNK', 'default')} B={B}: e2e {best * 1e3:.1f} ms "
      f"{int(out['converged'].sum()) / best:.0f} flows/s", flush=True)
