"""Generate the golden vectors under tests/golden/ by running the REAL reference.

Runs only in the build container (needs /root/reference, read-only):

    PYTHONDONTWRITEBYTECODE=1 python tools/make_golden.py [--ref /root/reference/pkg/src]

Everything is produced through the reference's own public API (acpflow
__init__.py): its loaders, model builders, ScenarioSpec/make_scenarios
(Philox multipliers), newton_solve (GMRES-FD Newton) and zbus_iterate. The
outputs are the parity anchors for oracle/ (CPU tests) and for the CUDA path
(GPU tests); nothing at run time reads /root/reference.
"""

from __future__ import annotations

import argparse
import gzip
import sys
import tempfile
import time
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


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    sys.path.insert(0, args.ref)
    import acpflow as ac
    from acpflow import distribution as dmod

    OUT.mkdir(parents=True, exist_ok=True)
    only = set(filter(None, args.only.split(",")))

    # eulv.json must be byte-identical to the reference generator's output
    tools = Path(args.ref).parent / "tools" / "make_dist_fixtures.py"
    if tools.exists() and (not only or "eulv" in only):
        import subprocess
        with tempfile.TemporaryDirectory() as td:
            subprocess.run([sys.executable, str(tools), td], check=True, capture_output=True,
                           env={"PYTHONPATH": args.ref, "PYTHONDONTWRITEBYTECODE": "1",
                                "PATH": "/usr/bin:/bin"})
            fresh = (Path(td) / "eulv.json").read_bytes()
        assert fresh == gzip.open(FIX / "eulv.json.gz").read(), "fixtures/eulv.json.gz is stale"
        print("eulv.json.gz verified against the reference generator")

    def want(tag):
        return not only or tag in only

    # ---------------- Philox multipliers (batch.py:45-60)
    if want("philox"):
        specs = [(1010, 0.2, 4, 3), (7070, 0.2, 5, 12), (10010, 0.2, 7, 2), (2**63 + 5, 0.1, 6, 4)]
        d = {}
        for k, (seed, spread, n, count) in enumerate(specs):
            spec = ac.ScenarioSpec(count=count, seed=seed, spread=spread)
            d[f"m{k}"] = ac.generate_load_multipliers(spec, n)
            d[f"spec{k}"] = np.array([seed % 2**64, count, n], dtype=np.uint64)
            d[f"spread{k}"] = np.array(spread)
        np.savez_compressed(OUT / "philox.npz", **d)

    # ---------------- Transmission NR
    tx_cases = [("case14", "case14.m", 1010, 64, True), ("case118", "case118.m", 1010, 64, True),
                ("case1354", "case1354pegase.m", 1010, 12, False),
                ("gb2224", "gb2224.m", 10010, 8, True)]
    for tag, fname, seed, count, keep_state in tx_cases:
        if not want(tag):
            continue
        t0 = time.time()
        net = ac.parse_matpower_case(_text(fname))
        model = ac.build_transmission_model(net)
        part = model.part
        yc = model.y.complex_csr()
        base = ac.transmission_base(net, part)
        spec = ac.ScenarioSpec(count=count, seed=seed, spread=0.2)
        mult = ac.generate_load_multipliers(spec, base.n_elements)
        scen = [ac.apply_multipliers(base, mult[i]) for i in range(count)]
        res = [ac.newton_solve(model, sc) for sc in scen]
        bsc = ac.base_scenario(net, part)
        bres = ac.newton_solve(model, bsc)
        huge = ac.TransmissionScenario(p_spec=50 * bsc.p_spec, q_spec=50 * bsc.q_spec)
        hres = ac.newton_solve(model, huge)
        st = ac.flat_start(net, part)
        d = dict(
            y_indptr=yc.indptr.astype(np.int64), y_indices=yc.indices.astype(np.int64), y_data=yc.data,
            theta_block=part.theta_block, q_block=part.q_block, slack=np.array(part.slack),
            theta0=st.theta, vmag0=st.vmag, load_elements=base.load_elements,
            seed=np.array(seed, dtype=np.uint64), multipliers=mult,
            p_spec=np.stack([s.p_spec for s in scen]), q_spec=np.stack([s.q_spec for s in scen]),
            converged=np.array([r.converged for r in res]),
            iterations=np.array([r.iterations for r in res]),
            fnorm=np.array([r.final_mismatch_inf for r in res]),
            gmres_total=np.array([r.total_gmres_iterations for r in res]),
            base_theta=bres.state.theta, base_vmag=bres.state.vmag,
            base_iterations=np.array(bres.iterations), base_fnorm=np.array(bres.final_mismatch_inf),
            huge_converged=np.array(hres.converged), huge_iterations=np.array(hres.iterations),
            huge_fnorm=np.array(hres.final_mismatch_inf),
            huge_diagnostic=np.array(hres.diagnostic or ""),
        )
        if keep_state:
            d["theta"] = np.stack([r.state.theta for r in res])
            d["vmag"] = np.stack([r.state.vmag for r in res])
        if tag in ("case14", "case118"):
            # a non-flat state and the reference's dense Jacobian there
            rng = np.random.default_rng(99)
            x = st.pack(part) + np.concatenate([rng.normal(scale=0.05, size=part.n_theta),
                                                rng.normal(scale=0.04, size=part.n_q)])
            s2 = st.with_packed(x, part)
            d["jac_theta"] = s2.theta
            d["jac_vmag"] = s2.vmag
            d["jac_dense"] = ac.dense_jacobian(s2, model.y, part)
            d["mis_at_state"] = ac.mismatch(s2, bsc, model.y, part)
        np.savez_compressed(OUT / f"nr_{tag}.npz", **d)
        print(f"{tag}: {count} scenarios, iterations {np.unique(d['iterations'])}, "
              f"all converged {d['converged'].all()}, {time.time() - t0:.1f}s")

    # ---------------- Distribution Z-Bus
    zb_cases = [("ieee13", "ieee13.json", 5050, 4096, 256), ("ieee123", "ieee123.json", 5050, 256, 32),
                ("eulv", "eulv.json", 10011, 64, 8)]
    for tag, fname, seed, count, keep_v in zb_cases:
        if not want(tag):
            continue
        t0 = time.time()
        net = ac.parse_distribution_json(_text(fname))
        model = ac.build_zbus_model(net)
        base = ac.distribution_base(model)
        spec = ac.ScenarioSpec(count=count, seed=seed, spread=0.2, target="distribution")
        mult = ac.generate_load_multipliers(spec, base.n_elements)
        scen = [ac.apply_multipliers(base, mult[i]) for i in range(count)]
        res = [ac.zbus_iterate(model, sc) for sc in scen]
        bres = ac.zbus_iterate(model)
        y = ac.build_three_phase_ybus(net)
        d = dict(
            y_indptr=y.indptr.astype(np.int64), y_indices=y.indices.astype(np.int64), y_data=y.data,
            v0=model.v0, non_slack=model.non_slack, wye_idx=model.wye_idx, delta_p=model.delta_p,
            delta_q=model.delta_q, wye_s=model.wye_s, delta_s=model.delta_s,
            seed=np.array(seed, dtype=np.uint64), multipliers=mult,
            s_wye=np.stack([s.wye_s for s in scen]), s_delta=np.stack([s.delta_s for s in scen]),
            converged=np.array([r.converged for r in res]),
            iterations=np.array([r.iterations for r in res]),
            final_delta=np.array([r.final_delta for r in res]),
            residual=np.array([r.residual_inf for r in res]),
            v=np.stack([r.v for r in res[:keep_v]]),
            base_v=bres.v, base_iterations=np.array(bres.iterations),
            base_final_delta=np.array(bres.final_delta), base_residual=np.array(bres.residual_inf),
        )
        if tag == "ieee13":
            cols = np.unique(np.concatenate([model.wye_idx, model.delta_p, model.delta_q]))
            e = np.zeros((model.n, cols.size), dtype=complex)
            e[cols, np.arange(cols.size)] = 1.0
            d["z_load"] = np.stack([model.z_apply(e[:, k]) for k in range(cols.size)], axis=1)
            d["load_cols"] = cols
            # no-load scenario and a 500x divergent one (tests/test_distribution.py:303, :351)
            zr = ac.zbus_iterate(model, dmod.DistributionScenario(np.zeros_like(model.wye_s),
                                                                  np.zeros_like(model.delta_s)))
            d["noload_v"] = zr.v
            d["noload_iterations"] = np.array(zr.iterations)
            hv = ac.zbus_iterate(model, dmod.DistributionScenario(model.wye_s * 60.0, model.delta_s * 60.0))
            d["heavy_converged"] = np.array(hv.converged)
            d["heavy_iterations"] = np.array(hv.iterations)
            d["heavy_diagnostic"] = np.array(hv.diagnostic or "")
            d["heavy_final_delta"] = np.array(hv.final_delta)
            d["heavy_residual"] = np.array(hv.residual_inf)
            d["heavy_v"] = hv.v
        np.savez_compressed(OUT / f"zb_{tag}.npz", **d)
        print(f"{tag}: {count} scenarios, iterations {np.unique(d['iterations'], return_counts=True)}, "
              f"{time.time() - t0:.1f}s")
    return 0


if __name__ == "__main__":
    sys.exit(main())
