"""Per-step device time of the NR solve vs the library's own kernel time
(acpf_nr_last_timing): the gap is host work between the Newton steps."""
import sys
import time

import torch

sys.path.insert(0, '.')
import paper_2605_14103_b200 as pf  # noqa: E402
from paper_2605_14103_b200.fixtures import load_transmission  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
net = load_transmission('gb2224')
import os
m = pf.build_transmission_model(net, ordering=os.environ.get('ACPF_PROBE_ORDER', 'minfill'))
base = pf.transmission_base(net, m.part)
plan = m.plan()
pt, qt = plan.scenarios(base, 10010, 0, B, 0.2, device=0)
out = plan.alloc_outputs(B, like=pt)
st = torch.cuda.current_stream()
for k in range(int(sys.argv[2]) if len(sys.argv) > 2 else 8):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    h0 = time.perf_counter()
    e0.record(st)
    plan.solve(pt, qt, 1e-8, 20, out=out, stream=st)
    e1.record(st)
    torch.cuda.synchronize()
    h1 = time.perf_counter()
    print(f"step {k}: events {e0.elapsed_time(e1):.1f} ms, host {1e3 * (h1 - h0):.1f} ms, "
          f"kernel {plan.last_timing()[0]:.1f} ms, launches {plan.last_timing()[1]}", flush=True)
