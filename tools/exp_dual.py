"""Probe: do two half-batches on two streams overlap better than one batch?

    python tools/exp_dual.py [B]

(a) one plan, B scenarios, full solve; (b) two plans, B/2 each, solved from two
host threads on two streams concurrently; (c) one plan, B/2 twice in sequence.
Wall time around each with device synchronisation (probe only, not a bench).
"""
import sys
import threading
import time

import torch

sys.path.insert(0, '.')
import paper_2605_14103_b200 as pf  # noqa: E402
from paper_2605_14103_b200.fixtures import load_transmission  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
net = load_transmission('gb2224')
m = pf.build_transmission_model(net)
base = pf.transmission_base(net, m.part)
p1, p2 = m.plan(), pf.build_transmission_model(net).plan()
pt, qt = p1.scenarios(base, 10010, 0, B, 0.2, device=0)
h = B // 2
halves = [(pt[:h].contiguous(), qt[:h].contiguous()), (pt[h:].contiguous(), qt[h:].contiguous())]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
out_full = p1.solve(pt, qt, 1e-8, 20)
outs = [p1.solve(*halves[0], 1e-8, 20), p2.solve(*halves[1], 1e-8, 20)]


def timed(fn, reps=3):
    best = 1e30
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


def single():
    p1.solve(pt, qt, 1e-8, 20, out=out_full, stream=s1)


OFFSET = [0.0]  # seconds the second half starts after the first (phase offset)


def dual():
    def second():
        time.sleep(OFFSET[0])
        p2.solve(*halves[1], 1e-8, 20, out=outs[1], stream=s2)
    ths = [threading.Thread(target=lambda: p1.solve(*halves[0], 1e-8, 20, out=outs[0], stream=s1)),
           threading.Thread(target=second)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()


def seq():
    p1.solve(*halves[0], 1e-8, 20, out=outs[0], stream=s1)
    p1.solve(*halves[1], 1e-8, 20, out=outs[1], stream=s1)


for name, fn in (("single", single), ("dual", dual), ("seq-halves", seq), ("single", single), ("dual", dual)):
    t = timed(fn)
    print(f"{name:10s} B={B}: {t * 1e3:8.1f} ms  {B / t:9.0f} flows/s", flush=True)
for off in (0.010, 0.020, 0.040, 0.060):
    OFFSET[0] = off
    t = timed(dual)
    print(f"dual+{off * 1e3:.0f}ms B={B}: {t * 1e3:8.1f} ms  {B / t:9.0f} flows/s", flush=True)
conv = int(outs[0]["converged"].sum().item() + outs[1]["converged"].sum().item())
print("dual converged", conv, "single", int(out_full["converged"].sum().item()))
