"""Scale-level golden summaries from the REAL reference (build container only).

    PYTHONDONTWRITEBYTECODE=1 python tools/make_golden_scale.py [--ref /root/reference/pkg/src] [--sets a,b]

Solves seeded scenario sets through the reference's public API on a process
pool: NR with `newton_solve` -- 4,096 GBnetwork (seed 10010, the acceptance
seed; scale_nr_gb2224), 4,096 case1354pegase and 4,096 case118 (round 2) --
and Z-Bus with `zbus_iterate` -- 16,384 EULV (seed 10011; scale_zb_eulv),
16,384 IEEE123 and 16,384 IEEE13 (round 2). The
scenario inputs are not stored (they are the reference generator's rows
0..count-1, reproduced bitwise by the engine); stored are the per-scenario
flags, iteration counts, GMRES totals, residuals, fixed-order state summaries
the full state of every 64th scenario, and the decision margins of the stop
rules: the NR mismatch norm at every Newton check (recorded by wrapping
transmission.mismatch, result unchanged) and the Z-Bus |sum|v_k| - sum|v_k-1||
of every sweep (wrapping ZBusModel.z_apply, tools/make_golden_failures.py).
tests/test_gpu_scale.py / test_gpu_fullsize.py check the CUDA path against
them and report stop-rule ties (tests/tiebands.py) separately.
"""

from __future__ import annotations

import argparse
import gzip
import sys
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "tests" / "golden"
FIX = ROOT / "fixtures"
REF = "/root/reference/pkg/src"
KEEP_EVERY = 64
# set name -> (fixture, count, seed)
NR_SETS = {"gb2224": ("gb2224.m", 4096, 10010), "case1354": ("case1354pegase.m", 4096, 10010),
           "case118": ("case118.m", 4096, 10010)}
ZB_SETS = {"eulv": ("eulv.json", 16384, 10011), "ieee123": ("ieee123.json", 16384, 10011),
           "ieee13": ("ieee13.json", 16384, 10011)}

_state = {}


def _text(name: str) -> str:
    p = FIX / name
    if p.exists():
        return p.read_text()
    with gzip.open(str(p) + ".gz", "rt") as fh:
        return fh.read()


def _init(ref: str, kind: str, name: str):
    sys.path.insert(0, ref)
    sys.path.insert(0, str(ROOT / "tools"))
    import acpflow as ac
    from acpflow import distribution as dm
    from acpflow import transmission as tm
    from make_golden_failures import _DeltaRecorder
    _state["ac"] = ac
    rec = _DeltaRecorder(dm)
    rec.__enter__()
    _state["rec"] = rec
    orig = tm.mismatch
    _state["fn"] = None

    def mismatch(*a, **k):
        f = orig(*a, **k)
        if _state["fn"] is not None:
            _state["fn"].append(float(np.abs(f).max()) if f.size else 0.0)
        return f

    tm.mismatch = mismatch
    if kind == "nr":
        fname, count, seed = NR_SETS[name]
        net = ac.parse_matpower_case(_text(fname))
        model = ac.build_transmission_model(net)
        base = ac.transmission_base(net, model.part)
        mult = ac.generate_load_multipliers(ac.ScenarioSpec(count=count, seed=seed, spread=0.2), base.n_elements)
        _state["nr"] = (model, base, mult)
    else:
        fname, count, seed = ZB_SETS[name]
        dnet = ac.parse_distribution_json(_text(fname))
        dmodel = ac.build_zbus_model(dnet)
        dbase = ac.distribution_base(dmodel)
        dmult = ac.generate_load_multipliers(
            ac.ScenarioSpec(count=count, seed=seed, spread=0.2, target="distribution"), dbase.n_elements)
        _state["zb"] = (dmodel, dbase, dmult)


def _nr(i: int):
    ac = _state["ac"]
    model, base, mult = _state["nr"]
    _state["fn"] = []
    r = ac.newton_solve(model, ac.apply_multipliers(base, mult[i]))
    fn = _state["fn"]
    _state["fn"] = None
    return (r.converged, r.iterations, r.total_gmres_iterations, r.final_mismatch_inf, r.state.theta,
            r.state.vmag, fn)


def _zb(i: int):
    ac = _state["ac"]
    model, base, mult = _state["zb"]
    r, d = _state["rec"].run(ac, model, ac.apply_multipliers(base, mult[i]))
    return r.converged, r.iterations, r.final_delta, r.residual_inf, r.v, d


def _pad(seqs):
    m = max(len(x) for x in seqs)
    a = np.full((len(seqs), m), np.nan)
    for k, x in enumerate(seqs):
        a[k, :len(x)] = x
    return a


def _run_nr(name: str, ref: str, workers: int) -> None:
    fname, count, seed = NR_SETS[name]
    with ProcessPoolExecutor(workers, initializer=_init, initargs=(ref, "nr", name)) as ex:
        nr = list(ex.map(_nr, range(count), chunksize=8))
    keep = np.arange(0, count, KEEP_EVERY)
    th = np.array([r[4] for r in nr])
    vm = np.array([r[5] for r in nr])
    np.savez_compressed(
        OUT / f"scale_nr_{name}.npz", seed=seed, count=count,
        converged=np.array([r[0] for r in nr]), iterations=np.array([r[1] for r in nr]),
        gmres_total=np.array([r[2] for r in nr]), fnorm=np.array([r[3] for r in nr]),
        theta_sum=th.sum(1), vmag_sum=vm.sum(1), vmag_min=vm.min(1), vmag_max=vm.max(1),
        keep=keep, theta=th[keep], vmag=vm[keep], step_fnorm=_pad([r[6] for r in nr]))
    print(f"NR {name} iterations", np.unique([r[1] for r in nr], return_counts=True))


def _run_zb(name: str, ref: str, workers: int) -> None:
    fname, count, seed = ZB_SETS[name]
    with ProcessPoolExecutor(workers, initializer=_init, initargs=(ref, "zb", name)) as ex:
        zb = list(ex.map(_zb, range(count), chunksize=32))
    keepz = np.arange(0, count, KEEP_EVERY)
    v = np.array([r[4] for r in zb])
    np.savez_compressed(
        OUT / f"scale_zb_{name}.npz", seed=seed, count=count,
        converged=np.array([r[0] for r in zb]), iterations=np.array([r[1] for r in zb]),
        final_delta=np.array([r[2] for r in zb]), residual=np.array([r[3] for r in zb]),
        vabs_sum=np.abs(v).sum(1), vabs_min=np.abs(v).min(1), keep=keepz, v=v[keepz],
        sweep_delta=_pad([r[5] for r in zb]))
    print(f"ZB {name} iterations", np.unique([r[1] for r in zb], return_counts=True))


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default=REF)
    ap.add_argument("--workers", type=int, default=8)
    ap.add_argument("--sets", default=",".join(list(NR_SETS) + list(ZB_SETS)),
                    help="comma-separated set names (NR: gb2224, case1354, case118; Z-Bus: eulv, ieee123, ieee13)")
    args = ap.parse_args()
    for name in filter(None, args.sets.split(",")):
        if name in NR_SETS:
            _run_nr(name, args.ref, args.workers)
        elif name in ZB_SETS:
            _run_zb(name, args.ref, args.workers)
        else:
            raise SystemExit(f"unknown set {name!r}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
