"""Quick throughput probe (device-resident inputs, kernel time by CUDA events).

Scenarios are the seeded reference batch (distinct scenarios, no tiling); the
iteration histogram must match the reference (gb2224: 4, eulv: 10-12).
"""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_2605_14103_b200 as pf
from paper_2605_14103_b200 import engine
from paper_2605_14103_b200.fixtures import load_transmission, load_distribution

def gen(base, seed, count, target):
    return pf.make_scenario_arrays(base, pf.ScenarioSpec(count=count, seed=seed, target=target))

which = sys.argv[1] if len(sys.argv) > 1 else 'both'
if which in ('nr', 'both'):
    net = load_transmission('gb2224'); m = pf.build_transmission_model(net)
    plan = m.plan(); print(plan.info)
    base = pf.transmission_base(net, m.part)
    for B in [int(x) for x in (sys.argv[2].split(',') if len(sys.argv) > 2 else ['1024', '4096', '16384'])]:
        p, q = gen(base, 10010, B, 'transmission')
        pt, qt = torch.from_numpy(p).cuda(), torch.from_numpy(q).cuda()
        out = plan.solve(pt, qt, 1e-8, 20)
        torch.cuda.synchronize()
        plan.solve(pt, qt, 1e-8, 20, out=out); ms, nl = plan.last_timing()
        it = out['iterations'].cpu().numpy(); cv = out['converged'].cpu().numpy()
        print(f'NR gb2224 B={B}: kernel {ms:.2f} ms launches {nl} -> {B/ms*1e3:.0f} scen/s; iters {np.unique(it, return_counts=True)} conv {cv.mean()}', flush=True)
if which in ('zb', 'both'):
    net = load_distribution('eulv'); m = pf.build_zbus_model(net)
    plan = engine.zbus_plan_for(m)
    base = pf.distribution_base(m)
    for B in [int(x) for x in (sys.argv[3].split(',') if len(sys.argv) > 3 else ['4096', '16384', '65536'])]:
        sw, sd = gen(base, 10011, B, 'distribution')
        swt = torch.from_numpy(sw).cuda(); sdt = torch.from_numpy(sd.reshape(B, -1)).cuda()
        out = plan.solve(swt, sdt, 1e-9, 100)
        plan.solve(swt, sdt, 1e-9, 100, out=out); ms, nl = plan.last_timing()
        it = out['iterations'].cpu().numpy()
        print(f'ZB eulv B={B}: kernel {ms:.2f} ms -> {B/ms*1e3:.0f} scen/s; iters {np.unique(it, return_counts=True)}', flush=True)
