"""Golden vectors for the failure branches, from the REAL reference (build container only).

    PYTHONDONTWRITEBYTECODE=1 python tools/make_golden_failures.py [--ref /root/reference/pkg/src]

Every outcome is produced by the reference's public API (newton_solve,
zbus_iterate, build_zbus_model(voltage_floor=...), NewtonOptions,
FixedPointOptions); the inputs are stored beside the outcomes, so the GPU tests
(tests/test_gpu_failures.py) replay them through the C-ABI without the
reference. Branches covered (reference file:line):

NR `_newton_loop` (transmission.py:333-380), tests/golden/fail_nr.npz
  * non-finite mismatch at k = 0 (NaN, +inf, -inf specified injections), :350-352
  * `max_newton` exit with iterations = max_newton and the fnorm of the last
    check (max_newton = 1, 2), :358-359, :380
  * a looser tolerance (tol_mismatch = 1e-4), :353-354
  * heavy loads (x2 .. x30 of the base case): slow convergence (5, 7
    iterations) and V <= 0 collapses at iterations 1 .. 10, :355-357
  * an extreme injection (1e150) that collapses at iteration 1
  * warm starts (`start=`, flat_start=False; :306-330): from the base case's
    solution and from a perturbed flat start
Z-Bus `_zbus_loop` (distribution.py:653-687), tests/golden/fail_zb.npz
  * VoltageFloorError on a wye phase at sweep 1 (v = v0) and at sweep 5
    (v = previous iterate), on a delta phase, and on a delta line-to-line
    voltage (label "p-q"), distribution.py:583-606, :662-672
  * mixed batches: seeded scenarios under a floor that stops some of them at
    different sweeps while the rest converge (IEEE13, IEEE123)
  * `max_iter` exits (max_iter = 5), and a looser tolerance (1e-6)
  * the per-sweep sum-of-magnitudes deltas of every scenario (recorded by
    wrapping ZBusModel.z_apply without changing its result) for the stop-rule
    tie-band classifier (SURVEY.md hard part 5)
"""

from __future__ import annotations

import argparse
import gzip
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "tests" / "golden"
FIX = ROOT / "fixtures"


def _text(name: str) -> str:
    p = FIX / name
    if p.exists():
        return p.read_text()
    with gzip.open(str(p) + ".gz", "rt") as fh:
        return fh.read()


def _nr_cases(ac):
    out = {}
    for tag, fname, seed, count in [("case14", "case14.m", 1010, 8), ("case118", "case118.m", 1010, 16),
                                    ("case1354", "case1354pegase.m", 1010, 4), ("gb2224", "gb2224.m", 10010, 4)]:
        net = ac.parse_matpower_case(_text(fname))
        model = ac.build_transmission_model(net)
        part = model.part
        base = ac.transmission_base(net, part)
        mult = ac.generate_load_multipliers(ac.ScenarioSpec(count=count, seed=seed, spread=0.2),
                                            base.n_elements)
        seeded = [ac.apply_multipliers(base, mult[i]) for i in range(count)]
        b = ac.base_scenario(net, part)
        rows = []  # (p, q, tol, max_newton, label)
        for mx in (1, 2):
            rows += [(s.p_spec, s.q_spec, 1e-8, mx, f"max_newton={mx}") for s in seeded]
        rows += [(s.p_spec, s.q_spec, 1e-4, 20, "tol=1e-4") for s in seeded]
        if tag == "case1354":
            for sc in (2, 4, 8, 30):
                rows.append((sc * b.p_spec, sc * b.q_spec, 1e-8, 20, f"base x{sc}"))
        elif tag != "gb2224":
            for val, lab in ((np.nan, "nan"), (np.inf, "+inf"), (-np.inf, "-inf")):
                p = b.p_spec.copy()
                p[len(p) // 2] = val
                rows.append((p, b.q_spec, 1e-8, 20, f"p_spec {lab}"))
            q = b.q_spec.copy()
            q[0] = np.inf
            rows.append((b.p_spec, q, 1e-8, 20, "q_spec +inf"))
            for s in (2, 3, 4, 5, 6, 8, 10, 12, 15, 20, 30):
                rows.append((s * b.p_spec, s * b.q_spec, 1e-8, 20, f"base x{s}"))
            p = b.p_spec.copy()
            p[0] = 1e150
            rows.append((p, b.q_spec, 1e-8, 20, "p_spec[0] = 1e150"))
        # warm starts (transmission.py:306-330 `start=`): from the base case's
        # solution, and from a perturbed flat start, with flat_start=False
        flat = ac.flat_start(net, part)
        bsol = ac.newton_solve(model, b).state
        rng = np.random.default_rng(77)
        pert = ac.PolarState(flat.theta + rng.normal(scale=0.02, size=flat.theta.size),
                             flat.vmag * (1 + rng.normal(scale=0.01, size=flat.vmag.size)))
        starts = [None] * len(rows)
        for s in seeded[:4]:
            rows.append((s.p_spec, s.q_spec, 1e-8, 20, "warm: base solution"))
            starts.append(bsol)
            rows.append((s.p_spec, s.q_spec, 1e-8, 20, "warm: perturbed flat start"))
            starts.append(pert)
        res = []
        for (p, q, tol, mx, _), st in zip(rows, starts):
            opts = ac.NewtonOptions(tol_mismatch=tol, max_newton=mx, flat_start=st is None)
            res.append(ac.newton_solve(model, ac.TransmissionScenario(p, q), opts, start=st))
        th0 = np.stack([(flat if st is None else st).theta for st in starts])
        vm0 = np.stack([(flat if st is None else st).vmag for st in starts])
        out[tag] = dict(
            p_spec=np.stack([r[0] for r in rows]), q_spec=np.stack([r[1] for r in rows]),
            tol=np.array([r[2] for r in rows]), max_newton=np.array([r[3] for r in rows], dtype=np.int32),
            label=np.array([r[4] for r in rows]),
            converged=np.array([r.converged for r in res]), iterations=np.array([r.iterations for r in res]),
            fnorm=np.array([r.final_mismatch_inf for r in res]),
            diagnostic=np.array([r.diagnostic or "" for r in res]),
            theta=np.stack([r.state.theta for r in res]), vmag=np.stack([r.state.vmag for r in res]),
            has_start=np.array([st is not None for st in starts]), theta0=th0, vmag0=vm0)
        print(tag, [(r[4], x.converged, x.iterations, x.diagnostic) for r, x in zip(rows, res)
                    if not r[4].startswith(("max_newton", "tol"))])
    return out


class _DeltaRecorder:
    """Wraps ZBusModel.z_apply to record the loop's per-sweep |sum|v| - sum|v_prev||
    with the same numpy operations as distribution.py:673-676 (result unchanged)."""

    def __init__(self, dm):
        self.dm = dm
        self.orig = dm.ZBusModel.z_apply
        self.log = None

    def __enter__(self):
        rec = self

        def z_apply(model, w):
            x = rec.orig(model, w)
            if rec.log is not None:
                rec.log.append(float(np.abs(x + model.v0).sum()))
            return x

        self.dm.ZBusModel.z_apply = z_apply
        return self

    def __exit__(self, *a):
        self.dm.ZBusModel.z_apply = self.orig

    def run(self, ac, model, sc, opts=None):
        self.log = [float(np.abs(model.v0).sum())]
        r = ac.zbus_iterate(model, sc, opts)
        sums = self.log[: r.iterations + 1]  # the residual certificate's extra apply is dropped
        self.log = None
        return r, np.abs(np.diff(np.array(sums)))


def _zb_cases(ac, dm):
    ieee13 = _text("ieee13.json")
    doc = json.loads(ieee13)
    all_delta = dict(doc, loads=[ld for ld in doc["loads"] if ld["kind"] == "delta"])
    close_ab = json.loads(json.dumps(all_delta))
    a = close_ab["slack"]["voltage"]["a"]
    close_ab["slack"]["voltage"]["b"] = [a[0] * 0.999, a[1] + 0.0005]  # phases a, b nearly equal
    nets = {"ieee13": ieee13, "ieee13_all_delta": json.dumps(all_delta),
            "ieee13_close_ab": json.dumps(close_ab), "eulv": _text("eulv.json")}
    out = {}
    with _DeltaRecorder(dm) as rec:
        def solve_set(key, net_text, floor, scen, tol, max_iter, labels):
            net = ac.parse_distribution_json(net_text)
            model = ac.build_zbus_model(net, voltage_floor=floor)
            opts = dm.FixedPointOptions(tol=tol, max_iter=max_iter)
            res, deltas = [], []
            for sc in scen:
                r, d = rec.run(ac, model, sc, opts)
                res.append(r)
                deltas.append(d)
            kmax = max(len(d) for d in deltas)
            dl = np.full((len(res), max(kmax, 1)), np.nan)
            for k, d in enumerate(deltas):
                dl[k, :len(d)] = d
            out[key] = dict(
                network=np.array(net_text), floor=np.array(floor), tol=np.array(tol),
                max_iter=np.array(max_iter), label=np.array(labels),
                s_wye=np.stack([s.wye_s for s in scen]), s_delta=np.stack([s.delta_s for s in scen]),
                converged=np.array([r.converged for r in res]), iterations=np.array([r.iterations for r in res]),
                final_delta=np.array([r.final_delta for r in res]),
                residual=np.array([r.residual_inf for r in res]),
                diagnostic=np.array([r.diagnostic or "" for r in res]),
                v=np.stack([r.v for r in res]), sweep_delta=dl)
            print(key, [(lab, r.converged, r.iterations, r.diagnostic) for lab, r in zip(labels, res)][:8])
            return model

        base13 = ac.build_zbus_model(ac.parse_distribution_json(ieee13))
        b13 = dm.DistributionScenario(base13.wye_s, base13.delta_s)
        wmin0 = float(np.abs(base13.v0[base13.wye_idx]).min())
        solve_set("wye_sweep1", ieee13, wmin0 * 1.0001, [b13], 1e-9, 100, ["wye floor at v0"])
        solve_set("wye_sweep5", ieee13, 0.8949612188587067, [b13], 1e-9, 100, ["wye floor mid-iteration"])
        md = ac.build_zbus_model(ac.parse_distribution_json(nets["ieee13_all_delta"]))
        solve_set("delta_phase", nets["ieee13_all_delta"], 1.2,
                  [dm.DistributionScenario(md.wye_s, md.delta_s)], 1e-9, 100, ["delta phase floor at v0"])
        solve_set("delta_phase_mid", nets["ieee13_all_delta"], 0.93,
                  [dm.DistributionScenario(md.wye_s, md.delta_s * 3.0)], 1e-9, 100,
                  ["delta phase floor mid-iteration"])
        mc = ac.build_zbus_model(ac.parse_distribution_json(nets["ieee13_close_ab"]))
        solve_set("delta_line", nets["ieee13_close_ab"], 1e-3,
                  [dm.DistributionScenario(mc.wye_s, mc.delta_s)], 1e-9, 100, ["delta line-to-line floor"])
        # seeded batches
        base = ac.distribution_base(base13)
        mult = ac.generate_load_multipliers(
            ac.ScenarioSpec(count=256, seed=5050, spread=0.2, target="distribution"), base.n_elements)
        seeded = [ac.apply_multipliers(base, mult[i]) for i in range(256)]
        solve_set("mixed_floor", ieee13, 0.905, seeded, 1e-9, 100, ["seeded, floor 0.905"] * 256)
        solve_set("max_iter5", ieee13, 1e-6, seeded[:64], 1e-9, 5, ["max_iter=5"] * 64)
        solve_set("tol1e-6", ieee13, 1e-6, seeded[:64], 1e-6, 100, ["tol=1e-6"] * 64)
        # IEEE123: a floor that stops part of a seeded batch, and max_iter
        i123 = _text("ieee123.json")
        m123 = ac.build_zbus_model(ac.parse_distribution_json(i123))
        b123 = ac.distribution_base(m123)
        mu = ac.generate_load_multipliers(
            ac.ScenarioSpec(count=64, seed=5050, spread=0.2, target="distribution"), b123.n_elements)
        s123 = [ac.apply_multipliers(b123, mu[i]) for i in range(64)]
        base_sol = ac.zbus_iterate(m123)
        fl = float(np.quantile(np.abs(base_sol.v), 0.02))  # below a few load voltages of some scenarios
        solve_set("ieee123_floor", i123, fl, s123, 1e-9, 100, ["seeded, floor at the 2% |v| quantile"] * 64)
        solve_set("ieee123_max_iter3", i123, 1e-6, s123[:16], 1e-9, 3, ["max_iter=3"] * 16)
        eu = ac.build_zbus_model(ac.parse_distribution_json(nets["eulv"]))
        eb = ac.distribution_base(eu)
        em = ac.generate_load_multipliers(
            ac.ScenarioSpec(count=16, seed=10011, spread=0.2, target="distribution"), eb.n_elements)
        solve_set("eulv_max_iter5", nets["eulv"], 1e-6, [ac.apply_multipliers(eb, em[i]) for i in range(16)],
                  1e-9, 5, ["max_iter=5"] * 16)
    return out


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    args = ap.parse_args()
    sys.path.insert(0, args.ref)
    import acpflow as ac
    from acpflow import distribution as dm

    OUT.mkdir(parents=True, exist_ok=True)
    nr = _nr_cases(ac)
    np.savez_compressed(OUT / "fail_nr.npz", **{f"{t}__{k}": v for t, d in nr.items() for k, v in d.items()})
    zb = _zb_cases(ac, dm)
    np.savez_compressed(OUT / "fail_zb.npz", **{f"{t}__{k}": v for t, d in zb.items() for k, v in d.items()})
    return 0


if __name__ == "__main__":
    sys.exit(main())
