"""One-factorisation timing probe for kernel experiments.

    ACPF_LIB=exp/libacpf_x.so python tools/exp_probe.py 65536

Runs the batched Newton solve with max_newton=1 (one mismatch, one
factorisation + substitution, one final mismatch) on the seeded gb2224 batch and
prints the kernel time; used to compare experimental builds of the same code.
"""
import os, sys
import torch
sys.path.insert(0, '.')
import paper_2605_14103_b200 as pf
from paper_2605_14103_b200 import engine
from paper_2605_14103_b200.fixtures import load_transmission

net = load_transmission('gb2224'); m = pf.build_transmission_model(net)
plan = m.plan()
base = pf.transmission_base(net, m.part)
for B in [int(x) for x in (sys.argv[1].split(',') if len(sys.argv) > 1 else ['65536'])]:
    p, q = pf.make_scenario_arrays(base, pf.ScenarioSpec(count=B, seed=10010, target='transmission'))
    pt, qt = torch.from_numpy(p).cuda(), torch.from_numpy(q).cuda()
    out = plan.solve(pt, qt, 1e-8, 1)
    best = 1e30
    for _ in range(3):
        plan.solve(pt, qt, 1e-8, 1, out=out)
        ms, nl = plan.last_timing()
        best = min(best, ms)
    print(f"{os.environ.get('ACPF_LIB', 'default')} B={B}: one-step solve {best:.2f} ms", flush=True)
