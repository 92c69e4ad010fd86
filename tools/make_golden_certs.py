"""Reference-run goldens for the on-device certificates.

Runs only in the build container (needs /root/reference, read-only):

    PYTHONDONTWRITEBYTECODE=1 python tools/make_golden_certs.py [--ref /root/reference/pkg/src]

At fixed states -- the reference's own converged states from tests/golden
and the same states perturbed (so the certificates are O(1e-3), not
rounding noise) -- it records what the REAL reference computes:

  NR (acpf_nr_certify): ||mismatch||inf (transmission.py:202-215), the
      branch loss sum(s_from + s_to).real (branch_flows, :453-481), the
      slack injection p_calc[slack] (calc_injections, :194-199) and the bus
      shunt loss, i.e. every term of the slack balance of the reference's
      test_transmission.py:398-416.
  Z-Bus (acpf_zbus_kirchhoff): kirchhoff_residual (distribution.py:624-630).

Output: tests/golden/cert.npz. Nothing at run time reads /root/reference.
"""

from __future__ import annotations

import argparse
import gzip
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "tests" / "golden"
FIX = ROOT / "fixtures"

NR = {"case118": ("case118.m", 64), "gb2224": ("gb2224.m", 8)}
ZB = {"ieee13": ("ieee13.json", 64), "ieee123": ("ieee123.json", 64), "eulv": ("eulv.json", 8)}


def _text(name: str) -> str:
    p = FIX / name
    if p.exists():
        return p.read_text()
    with gzip.open(str(p) + ".gz", "rt") as fh:
        return fh.read()


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    args = ap.parse_args()
    sys.path.insert(0, args.ref)
    import acpflow as ac
    from acpflow import distribution as dmod
    from acpflow import transmission as tmod

    out = {}
    rng = np.random.default_rng(2605)
    for tag, (fname, count) in NR.items():
        g = np.load(OUT / f"nr_{tag}.npz")
        net = ac.parse_matpower_case(_text(fname))
        model = ac.build_transmission_model(net)
        part = model.part
        slack = int(part.slack[0])
        th = np.concatenate([g["theta"][:count], g["theta"][:count]])
        vm = np.concatenate([g["vmag"][:count], g["vmag"][:count]])
        p = np.concatenate([g["p_spec"][:count], g["p_spec"][:count]])
        q = np.concatenate([g["q_spec"][:count], g["q_spec"][:count]])
        # second half: perturbed states (non-slack angles, PQ magnitudes)
        th[count:, part.theta_block] += 1e-3 * rng.standard_normal((count, part.theta_block.size))
        vm[count:, part.q_block] *= 1.0 + 1e-3 * rng.standard_normal((count, part.q_block.size))
        rec = {k: np.empty(2 * count) for k in ("mismatch_inf", "branch_loss", "p_slack", "shunt_loss")}
        for k in range(2 * count):
            st = tmod.PolarState(theta=th[k].copy(), vmag=vm[k].copy())
            sc = ac.TransmissionScenario(p_spec=p[k], q_spec=q[k])
            rec["mismatch_inf"][k] = np.abs(tmod.mismatch(st, sc, model.y, part)).max()
            s_from, s_to = tmod.branch_flows(net, st)
            rec["branch_loss"][k] = (s_from + s_to).sum().real
            p_calc, _ = tmod.calc_injections(st, model.y)
            rec["p_slack"][k] = p_calc[slack]
            rec["shunt_loss"][k] = sum(b.gs * st.vmag[i] ** 2 for i, b in enumerate(net.buses))
        out[f"nr_{tag}__theta"], out[f"nr_{tag}__vmag"] = th, vm
        out[f"nr_{tag}__p_spec"], out[f"nr_{tag}__q_spec"] = p, q
        for key, v in rec.items():
            out[f"nr_{tag}__{key}"] = v
        print(f"nr {tag}: {2 * count} states, mismatch_inf max {rec['mismatch_inf'].max():.3e}")
    for tag, (fname, count) in ZB.items():
        g = np.load(OUT / f"zb_{tag}.npz")
        net = ac.parse_distribution_json(_text(fname))
        model = ac.build_zbus_model(net)
        n = min(count, g["v"].shape[0])
        v = np.concatenate([g["v"][:n], g["v"][:n]])
        v[n:] *= 1.0 + 1e-3 * (rng.standard_normal(v[n:].shape) + 1j * rng.standard_normal(v[n:].shape))
        sw = np.concatenate([g["s_wye"][:n], g["s_wye"][:n]])
        sd = np.concatenate([g["s_delta"][:n], g["s_delta"][:n]])
        kcl = np.array([dmod.kirchhoff_residual(model, dmod.DistributionScenario(sw[k], sd[k]), v[k])
                        for k in range(2 * n)])
        out[f"zb_{tag}__v"], out[f"zb_{tag}__s_wye"], out[f"zb_{tag}__s_delta"] = v, sw, sd
        out[f"zb_{tag}__kirchhoff"] = kcl
        print(f"zb {tag}: {2 * n} states, kirchhoff max {kcl.max():.3e}")
    np.savez_compressed(OUT / "cert.npz", **out)
    print("wrote", OUT / "cert.npz")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
