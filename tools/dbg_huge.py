import sys; sys.path.insert(0,'.')
import numpy as np, paper_2605_14103_b200 as pf
from paper_2605_14103_b200.fixtures import load_transmission
for c in ['case14','case118']:
    m = pf.build_transmission_model(load_transmission(c))
    sc = pf.base_scenario(m.net, m.part)
    out = m.plan().solve(np.ascontiguousarray(50*sc.p_spec[None]), np.ascontiguousarray(50*sc.q_spec[None]), 1e-8, 20)
    print(c, {k: v[:1] if v.ndim == 1 else v[0, :5] for k, v in out.items()})
    out = m.plan().solve(np.ascontiguousarray(sc.p_spec[None]), np.ascontiguousarray(sc.q_spec[None]), 1e-8, 20)
    print(c, 'base', {k: v[:1] if v.ndim == 1 else v[0, :5] for k, v in out.items()})
