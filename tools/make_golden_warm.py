"""Warm-start scale golden from the REAL reference (build container only).

    PYTHONDONTWRITEBYTECODE=1 python tools/make_golden_warm.py [--ref /root/reference/pkg/src]

4,096 case1354pegase scenarios (seed 10010, spread 0.2, the reference
generator) each solved with newton_solve(..., NewtonOptions(flat_start=False),
start=PolarState) (transmission.py:306-330) from the base case's solution
perturbed per scenario: theta += 0.02 z at the non-slack buses, vmag *= 1 +
0.01 z' at the PQ buses (z, z' standard normal rows of
np.random.default_rng(2607), regenerated identically by
tests/test_gpu_stress.py::test_warm_start_4096_reference_scenarios).
Recorded: flags, iterations, the norm at every Newton check, final norms and
every 64th state.
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
COUNT, SEED, WSEED, KEEP_EVERY = 4096, 10010, 2607, 64
_st = {}


def warm_starts(theta, vmag, slack, pq, count=COUNT, seed=WSEED):
    """The per-scenario start states (shared with the GPU test)."""
    rng = np.random.default_rng(seed)
    z = rng.standard_normal((count, theta.size))
    z2 = rng.standard_normal((count, vmag.size))
    th = np.tile(theta, (count, 1))
    vm = np.tile(vmag, (count, 1))
    mask = np.ones(theta.size, bool)
    mask[list(slack)] = False
    th[:, mask] += 0.02 * z[:, mask]
    pqi = np.asarray(list(pq), dtype=np.int64)
    vm[:, pqi] *= 1.0 + 0.01 * z2[:, pqi]
    return th, vm


def _init(ref):
    sys.path.insert(0, ref)
    import acpflow as ac
    from acpflow import transmission as tm
    _st["ac"], _st["tm"] = ac, tm
    net = ac.parse_matpower_case(gzip.open(ROOT / "fixtures" / "case1354pegase.m.gz", "rt").read())
    model = ac.build_transmission_model(net)
    base = ac.transmission_base(net, model.part)
    bsol = ac.newton_solve(model, ac.base_scenario(net, model.part)).state
    th0, vm0 = warm_starts(bsol.theta, bsol.vmag, model.part.slack, model.part.pq)
    mult = ac.generate_load_multipliers(ac.ScenarioSpec(count=COUNT, seed=SEED, spread=0.2), base.n_elements)
    _st.update(model=model, base=base, mult=mult, th0=th0, vm0=vm0, bsol=bsol)
    orig = tm.mismatch
    _st["rec"] = None

    def mismatch(*a, **k):
        f = orig(*a, **k)
        if _st["rec"] is not None:
            _st["rec"].append(float(np.abs(f).max()) if f.size else 0.0)
        return f

    tm.mismatch = mismatch


def _solve(i):
    ac, tm = _st["ac"], _st["tm"]
    _st["rec"] = []
    sc = ac.apply_multipliers(_st["base"], _st["mult"][i])
    r = ac.newton_solve(_st["model"], sc, ac.NewtonOptions(flat_start=False),
                        start=tm.PolarState(theta=_st["th0"][i].copy(), vmag=_st["vm0"][i].copy()))
    rec, _st["rec"] = _st["rec"], None
    return r.converged, r.iterations, r.final_mismatch_inf, r.state.theta, r.state.vmag, rec


def _base(_):
    b = _st["bsol"]
    return b.theta, b.vmag


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    ap.add_argument("--workers", type=int, default=8)
    args = ap.parse_args()
    with ProcessPoolExecutor(args.workers, initializer=_init, initargs=(args.ref,)) as ex:
        res = list(ex.map(_solve, range(COUNT), chunksize=8))
        base_theta, base_vmag = next(ex.map(_base, [0]))
    m = max(len(r[5]) for r in res)
    steps = np.full((COUNT, m), np.nan)
    for k, r in enumerate(res):
        steps[k, :len(r[5])] = r[5]
    keep = np.arange(0, COUNT, KEEP_EVERY)
    np.savez_compressed(OUT / "warm_nr_case1354.npz", seed=SEED, wseed=WSEED, count=COUNT,
                        base_theta=base_theta, base_vmag=base_vmag,
                        converged=np.array([r[0] for r in res]), iterations=np.array([r[1] for r in res]),
                        fnorm=np.array([r[2] for r in res]), step_fnorm=steps, keep=keep,
                        theta=np.array([res[k][3] for k in keep]), vmag=np.array([res[k][4] for k in keep]))
    import collections
    print("converged", collections.Counter(r[0] for r in res), "iterations",
          sorted(collections.Counter(r[1] for r in res).items()))
    return 0


if __name__ == "__main__":
    sys.exit(main())
