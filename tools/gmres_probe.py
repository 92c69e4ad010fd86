"""Throughput of the GMRES-FD ablation step vs the exact-LU step (gb2224).

    python tools/gmres_probe.py [batch ...]
"""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_2605_14103_b200 as pf
from paper_2605_14103_b200.fixtures import load_transmission

net = load_transmission('gb2224'); m = pf.build_transmission_model(net)
plan = m.plan()
plan.set_fd(m.y.csr, m.part.theta_block, m.part.q_block, 1e-6)
base = pf.transmission_base(net, m.part)
for B in [int(x) for x in (sys.argv[1:] or ['4096', '16384'])]:
    p, q = pf.make_scenario_arrays(base, pf.ScenarioSpec(count=B, seed=10010))
    pt, qt = torch.from_numpy(p).cuda(), torch.from_numpy(q).cuda()
    plan.solve_gmres(pt, qt, 1e-8, 20)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = plan.solve_gmres(pt, qt, 1e-8, 20)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    it = out['iterations'].cpu().numpy(); gs = out['gmres_steps'].cpu().numpy().sum(1)
    plan.solve(pt, qt, 1e-8, 20)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    o2 = plan.solve(pt, qt, 1e-8, 20)
    torch.cuda.synchronize()
    tl = time.perf_counter() - t1
    print(f"gb2224 B={B}: GMRES-FD {B / t:.0f} scen/s ({t * 1e3:.0f} ms; Newton its {np.unique(it)}, "
          f"GMRES its/scenario {gs.mean():.1f}) | exact LU {B / tl:.0f} scen/s; conv {out['converged'].float().mean().item()}",
          flush=True)
