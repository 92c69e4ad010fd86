"""Run one solve for profiling: python tools/profile_case.py nr|zb BATCH [reps]"""
import sys
import numpy as np
sys.path.insert(0, '.')
import torch
import paper_2605_14103_b200 as pf
from paper_2605_14103_b200 import engine
from paper_2605_14103_b200.fixtures import load_transmission, load_distribution

kind, B = sys.argv[1], int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
if kind == 'nr':
    net = load_transmission(sys.argv[4] if len(sys.argv) > 4 else 'gb2224')
    m = pf.build_transmission_model(net)
    base = pf.transmission_base(net, m.part)
    p, q = pf.make_scenario_arrays(base, pf.ScenarioSpec(count=B, seed=10010))
    pt, qt = torch.from_numpy(p).cuda(), torch.from_numpy(q).cuda()
    plan = m.plan()
    for _ in range(reps):
        out = plan.solve(pt, qt, 1e-8, 20)
    print('nr', plan.last_timing(), out['iterations'][:4].tolist())
else:
    net = load_distribution(sys.argv[4] if len(sys.argv) > 4 else 'eulv')
    m = pf.build_zbus_model(net)
    base = pf.distribution_base(m)
    sw, sd = pf.make_scenario_arrays(base, pf.ScenarioSpec(count=B, seed=10011, target='distribution'))
    plan = engine.zbus_plan_for(m)
    swt = torch.from_numpy(sw).cuda(); sdt = torch.from_numpy(np.ascontiguousarray(sd.reshape(B, -1))).cuda()
    for _ in range(reps):
        out = plan.solve(swt, sdt, 1e-9, 100)
    print('zb', plan.last_timing(), out['iterations'][:4].tolist())
