import sys
sys.path.insert(0, '.')
from paper_2605_14103_b200 import engine
engine._lib = engine.load_library('paper_2605_14103_b200/libacpf_prof.so')
import numpy as np, torch
import paper_2605_14103_b200 as pf
from paper_2605_14103_b200.fixtures import load_transmission
net = load_transmission(sys.argv[1] if len(sys.argv) > 1 else 'gb2224')
m = pf.build_transmission_model(net)
base = pf.transmission_base(net, m.part)
B = int(sys.argv[2]) if len(sys.argv) > 2 else 64
p, q = pf.make_scenario_arrays(base, pf.ScenarioSpec(count=B, seed=10010))
plan = m.plan()
print(plan.info)
out = plan.solve(torch.from_numpy(p).cuda(), torch.from_numpy(q).cuda(), 1e-8, 20)
torch.cuda.synchronize()
print('ms', plan.last_timing())
