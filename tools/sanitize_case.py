"""Small solves for compute-sanitizer: NR case118 x 40 and Z-Bus IEEE123 x 40."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2605_14103_b200 as pf
from paper_2605_14103_b200 import engine
from paper_2605_14103_b200.fixtures import load_transmission, load_distribution
net = load_transmission('case118'); m = pf.build_transmission_model(net)
p, q = pf.make_scenario_arrays(pf.transmission_base(net, m.part), pf.ScenarioSpec(count=40, seed=1010))
out = m.plan().solve(p, q, 1e-8, 20)
print('nr', out['converged'].all(), np.unique(out['iterations']))
zm = pf.build_zbus_model(load_distribution('ieee123'))
sw, sd = pf.make_scenario_arrays(pf.distribution_base(zm), pf.ScenarioSpec(count=40, seed=5050, target='distribution'))
zo = engine.zbus_solve_arrays(zm, sw, sd, 1e-9, 100)
print('zb', zo['converged'].all(), np.unique(zo['iterations']))
