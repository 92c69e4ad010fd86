"""A/B probe: solve the seeded gb2224 batch with the library ACPF_LIB points at,
print the one-step and full-solve kernel times, and save or compare the states.

    python tools/exp_ab.py save OUT.npz [B]      # reference build
    ACPF_LIB=exp/x.so python tools/exp_ab.py cmp OUT.npz [B]
"""
import os
import sys

import numpy as np

sys.path.insert(0, '.')
import paper_2605_14103_b200 as pf  # noqa: E402
from paper_2605_14103_b200.fixtures import load_transmission  # noqa: E402

mode, path = sys.argv[1], sys.argv[2]
B = int(sys.argv[3]) if len(sys.argv) > 3 else 65536
net = load_transmission('gb2224')
m = pf.build_transmission_model(net)
base = pf.transmission_base(net, m.part)
plan = m.plan()
pt, qt = plan.scenarios(base, 10010, 0, B, 0.2, device=0)
out = plan.solve(pt, qt, 1e-8, 20)
one = min((plan.solve(pt, qt, 1e-8, 1), plan.last_timing()[0])[1] for _ in range(3))
full = min((plan.solve(pt, qt, 1e-8, 20, out=out), plan.last_timing()[0])[1] for _ in range(3))
th, vm = out['theta'].cpu().numpy(), out['vmag'].cpu().numpy()
it = out['iterations'].cpu().numpy()
print(f"{os.environ.get('ACPF_LIB', 'default')}: one-step {one:.2f} ms, full solve {full:.2f} ms "
      f"({B / full * 1e3:.0f}/s), iterations {np.unique(it, return_counts=True)}", flush=True)
if mode == 'save':
    np.savez(path, th=th, vm=vm, it=it)
else:
    ref = np.load(path)
    print("bitwise theta", np.array_equal(th.view(np.uint64), ref['th'].view(np.uint64)),
          "vmag", np.array_equal(vm.view(np.uint64), ref['vm'].view(np.uint64)),
          "iters", np.array_equal(it, ref['it']), "max|dth|", float(np.abs(th - ref['th']).max()))
