"""Stress-batch golden from the REAL reference (build container only).

    PYTHONDONTWRITEBYTECODE=1 python tools/make_golden_stress.py [--ref /root/reference/pkg/src]

4,096 case118 scenarios whose outcomes are mixed inside one batch: the
reference generator's rows at spread 0.9 (seed 2605, batch.py:45-60,
apply_multipliers :121-159), each scaled by a stored factor f_k in [1, 4)
(p_spec * f_k, q_spec * f_k, as tools/make_golden_failures.py scales the
base). Solved with the reference's newton_solve: converged in 3-14
iterations, `max_newton` exits and V <= 0 collapses side by side, so the GPU
batch has to keep every scenario's own exit while its groups run on
(tests/test_gpu_stress.py). Recorded: flags, iterations, diagnostics, final
norms, the norm at every Newton check (stop-rule tie bands) and full states of
every 32nd scenario.

Z-Bus: 16,384 IEEE13 scenarios at spread 0.9 (seed 2606) scaled by factors in
[1, 2.2): ~80% converge after 11-60+ sweeps, the rest run to max_iter = 100 --
long runs with many stop decisions (recorded: |sum|v_k| - sum|v_k-1|| of every
sweep, as tools/make_golden_scale.py), flags, iterations, final deltas and v
of every 64th scenario.
"""

from __future__ import annotations

import argparse
import gzip
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "tests" / "golden"
COUNT, SEED, SPREAD, KEEP_EVERY = 4096, 2605, 0.9, 32


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    args = ap.parse_args()
    sys.path.insert(0, args.ref)
    import acpflow as ac
    from acpflow import transmission as tm
    txt = gzip.open(ROOT / "fixtures" / "case118.m.gz", "rt").read()
    net = ac.parse_matpower_case(txt)
    model = ac.build_transmission_model(net)
    base = ac.transmission_base(net, model.part)
    mult = ac.generate_load_multipliers(ac.ScenarioSpec(count=COUNT, seed=SEED, spread=SPREAD), base.n_elements)
    factor = 1.0 + 3.0 * np.random.default_rng(SEED).random(COUNT)
    orig = tm.mismatch
    rec = []

    def mismatch(*a, **k):
        f = orig(*a, **k)
        rec.append(float(np.abs(f).max()) if f.size else 0.0)
        return f

    tm.mismatch = mismatch
    conv, its, diag, fnorm, steps, th, vm = [], [], [], [], [], [], []
    for i in range(COUNT):
        sc = ac.apply_multipliers(base, mult[i])
        sc = ac.TransmissionScenario(p_spec=sc.p_spec * factor[i], q_spec=sc.q_spec * factor[i])
        rec.clear()
        r = ac.newton_solve(model, sc)
        conv.append(r.converged)
        its.append(r.iterations)
        diag.append(r.diagnostic or "")
        fnorm.append(r.final_mismatch_inf)
        steps.append(list(rec))
        th.append(r.state.theta)
        vm.append(r.state.vmag)
    tm.mismatch = orig
    m = max(len(x) for x in steps)
    step_fnorm = np.full((COUNT, m), np.nan)
    for k, x in enumerate(steps):
        step_fnorm[k, :len(x)] = x
    keep = np.arange(0, COUNT, KEEP_EVERY)
    np.savez_compressed(OUT / "stress_nr_case118.npz", seed=SEED, spread=SPREAD, count=COUNT, factor=factor,
                        converged=np.array(conv), iterations=np.array(its), diagnostic=np.array(diag),
                        fnorm=np.array(fnorm), step_fnorm=step_fnorm, keep=keep,
                        theta=np.array(th)[keep], vmag=np.array(vm)[keep])
    import collections
    print("converged", collections.Counter(conv), "iterations", sorted(collections.Counter(its).items()))
    print("diagnostics", collections.Counter(d[:40] for d in diag).most_common(5))
    _zbus(ac)
    return 0


def _zbus(ac) -> None:
    from acpflow import distribution as dm
    sys.path.insert(0, str(ROOT / "tools"))
    from make_golden_failures import _DeltaRecorder
    count, seed, spread, lo, hi = 16384, 2606, 0.9, 1.0, 2.2
    txt = gzip.open(ROOT / "fixtures" / "ieee13.json.gz", "rt").read()
    model = ac.build_zbus_model(ac.parse_distribution_json(txt))
    base = ac.distribution_base(model)
    mult = ac.generate_load_multipliers(ac.ScenarioSpec(count=count, seed=seed, spread=spread,
                                                        target="distribution"), base.n_elements)
    factor = lo + (hi - lo) * np.random.default_rng(seed).random(count)
    conv, its, fdel, resid, vs, deltas = [], [], [], [], [], []
    with _DeltaRecorder(dm) as rec:
        for i in range(count):
            sc = ac.apply_multipliers(base, mult[i])
            sc = dm.DistributionScenario(sc.wye_s * factor[i], sc.delta_s * factor[i])
            r, d = rec.run(ac, model, sc)
            conv.append(r.converged)
            its.append(r.iterations)
            fdel.append(r.final_delta)
            resid.append(r.residual_inf)
            vs.append(r.v)
            deltas.append(d)
    m = max(len(x) for x in deltas)
    sweep = np.full((count, m), np.nan)
    for k, x in enumerate(deltas):
        sweep[k, :len(x)] = x
    keep = np.arange(0, count, 64)
    np.savez_compressed(OUT / "stress_zb_ieee13.npz", seed=seed, spread=spread, count=count, factor=factor,
                        converged=np.array(conv), iterations=np.array(its), final_delta=np.array(fdel),
                        residual=np.array(resid), sweep_delta=sweep, keep=keep, v=np.array(vs)[keep])
    import collections
    print("Z-Bus converged", collections.Counter(conv), "iterations (min, max, #100)",
          min(its), max(its), sum(1 for x in its if x == 100))


if __name__ == "__main__":
    sys.exit(main())
