"""Command-line driver routed onto the GPU engine (reference ``cli.py``).

    python -m paper_2605_14103_b200.cli solve  --case gb2224 --batch 4096 --seed 10010
    python -m paper_2605_14103_b200.cli bench  --case eulv --batch 65536
    python -m paper_2605_14103_b200.cli verify --case ieee13

Same subcommands, flags and exit-code contract as the reference (cli.py:26-28,
312-329): 0 ok, 1 input error, 2 numerical non-convergence / verification
failure. ``--case`` is a file path or a fixture name. Scenarios are generated
on the device (bitwise the reference generator). ``verify`` checks the GPU
solution with certificates computed on the device (NR: ||F||inf and the
slack power balance at the returned state, acpf_nr_certify; Z-Bus: the
reference CSV profile within 1e-3, as the reference does, plus the Kirchhoff
residual, acpf_zbus_kirchhoff).
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

from . import batch as bm
from . import distribution as dm
from . import engine
from . import network as nm
from . import transmission as tm
from .fixtures import FIXTURES, read_fixture

EXIT_OK, EXIT_INPUT, EXIT_NUMERICAL = 0, 1, 2
BENCH_SIZES = (1, 8, 64, 256, 1024, 4096, 16384, 65536)


class CliInputError(ValueError):
    def __init__(self, code: str, message: str):
        self.code = code
        super().__init__(message)


def _text(case: str) -> tuple:
    p = Path(case)
    if p.exists():
        return str(p), p.read_text(encoding="utf-8")
    for name in (case, case + ".m", case + ".json"):
        try:
            return name, read_fixture(name)
        except FileNotFoundError:
            continue
    raise CliInputError("io", f"no such file or fixture: {case}")


def _kind(path: str, kind: str | None, text: str) -> str:
    if kind:
        return kind
    if path.endswith(".m"):
        return "tx"
    if path.endswith(".json"):
        schema = json.loads(text).get("schema", "")
        if schema == dm.ZBUS_SCHEMA:
            return "dist"
        if schema == nm.TXNET_SCHEMA:
            return "tx"
    raise CliInputError("input", f"{path}: cannot infer network kind; pass --kind")


def _load(args):
    path, text = _text(args.case)
    kind = _kind(path, args.kind, text)
    if kind == "tx":
        net = nm.network_from_json(text) if path.endswith(".json") else nm.parse_matpower_case(text)
        model = tm.build_transmission_model(net)
        base = bm.transmission_base(net, model.part)
    else:
        net = dm.parse_distribution_json(text)
        model = dm.build_zbus_model(net)
        base = bm.distribution_base(model)
    return path, kind, model, base


def _solve_device(kind, model, base, seed, count, spread, tol, step="lu", precond="fd"):
    """Generate and solve `count` seeded scenarios on the device; host results.
    ``step`` "gmres" runs the reference's GMRES step (``precond`` fd|none)."""
    import torch
    dev = torch.device("cuda", 0)
    if kind == "tx":
        plan = model.plan(0)
        p, q = plan.scenarios(base, seed, 0, count, spread, device=dev)
        if step == "gmres":
            plan.set_fd(model.y.csr, model.part.theta_block, model.part.q_block, 1e-6)
        t0 = time.perf_counter()
        if step == "gmres":
            out = plan.solve_gmres(p, q, tol if tol is not None else 1e-8, 20, precond=precond)
        else:
            out = plan.solve(p, q, tol if tol is not None else 1e-8, 20)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    else:
        plan = engine.zbus_plan_for(model, 0)
        sw, sd = plan.scenarios(base, seed, 0, count, spread, device=dev)
        t0 = time.perf_counter()
        out = plan.solve(sw, sd, tol if tol is not None else 1e-9, 100)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    return {k: v.cpu().numpy() for k, v in out.items()}, wall


def cmd_solve(args) -> int:
    """`solve`: the device batch, then the acpflow-solve-result/1 document
    (or the report CSV) written natively from the result arrays
    (engine.solve_result_json / report_csv; reference cli.py:100-180)."""
    from .results import NewtonResults, ZbusResults
    path, kind, model, base = _load(args)
    out, wall = _solve_device(kind, model, base, args.seed, args.batch, args.spread, args.tol, args.step,
                              args.precond)
    res = NewtonResults(out) if kind == "tx" else ZbusResults(model, out)
    n = len(res)
    conv, its, resid, diag = res.converged(), res.iterations(), res.residuals(), res.diagnostics()
    if args.verbose:
        print(f"{int(conv.sum())}/{n} converged in {wall:.3f}s on the GPU", file=sys.stderr)
    share = wall / n
    # no --out: the native writer streams to stdout (the document of a large
    # batch never exists as one Python string)
    target = args.out
    if target is None:
        try:  # a real descriptor (not an in-process redirect such as a test's capture)
            fd = sys.stdout.fileno()
        except (AttributeError, OSError, ValueError):
            fd = None
        if fd is not None and Path(f"/dev/fd/{fd}").exists():
            sys.stdout.flush()
            target = f"/dev/fd/{fd}"
    if args.format == "csv":
        payload = engine.report_csv(conv, its, resid, share, diag, path=target)
    else:
        meta = {"case": Path(path).name, "kind": kind, "seed": args.seed, "spread": args.spread,
                "batch": args.batch, "worker_count": 1, "total_wall_time": wall,
                "throughput": n / wall if wall > 0 else float("inf")}
        if kind == "tx":
            a, b, ids = out["theta"], out["vmag"], None
        else:
            v = np.asarray(out["v"])
            a, b, ids = np.ascontiguousarray(v.real), np.ascontiguousarray(v.imag), model.reduced_ids()
        payload = engine.solve_result_json(meta, conv, its, resid, share, diag, a, b,
                                           node_phase_ids=ids, path=target)
    if payload is not None:
        sys.stdout.write(payload)
    return EXIT_OK if bool(conv.all()) else EXIT_NUMERICAL


def cmd_bench(args) -> int:
    path, kind, model, base = _load(args)
    top = args.batch if args.batch > 1 else 16384
    sizes = [s for s in BENCH_SIZES if s <= top] or [top]
    if top not in sizes:
        sizes.append(top)
    lines = ["case,kind,batch_size,workers,n_converged,total_wall_time,throughput"]
    _solve_device(kind, model, base, args.seed, 1, args.spread, args.tol, args.step, args.precond)  # warm-up
    for size in sizes:
        out, wall = _solve_device(kind, model, base, args.seed, size, args.spread, args.tol, args.step,
                                  args.precond)
        lines.append(f"{Path(path).name},{kind},{size},1,{int(out['converged'].sum())},{wall!r},"
                     f"{size / wall!r}")
    payload = "\n".join(lines) + "\n"
    if args.out:
        Path(args.out).write_text(payload, encoding="utf-8")
    else:
        sys.stdout.write(payload)
    return EXIT_OK


def cmd_verify(args) -> int:
    path, kind, model, base = _load(args)
    if kind == "tx":
        tol = args.tol if args.tol is not None else 1e-10
        res = tm.newton_solve(model, opts=tm.NewtonOptions(tol_mismatch=1e-10))
        sc = tm.base_scenario(model.net, model.part)
        # certificates computed on the device (acpf_nr_certify)
        plan = model.plan()
        plan.set_branches(model.net)
        cert = plan.certify(res.state.theta[None, :].copy(), res.state.vmag[None, :].copy(),
                            np.ascontiguousarray(sc.p_spec[None, :]), np.ascontiguousarray(sc.q_spec[None, :]))
        fn = float(cert["mismatch_inf"][0])
        bal = float(cert["slack_balance"][0])
        print("quantity                     value")
        print(f"||F||inf at GPU solution     {fn:.3e}  (threshold {tol:.1e})")
        print(f"slack power balance          {bal:.3e}  (threshold 1.0e-08)")
        print(f"branch loss (p.u.)           {float(cert['branch_loss'][0]):.6f}")
        print(f"solver converged             {res.converged}")
        return EXIT_OK if res.converged and fn <= tol and abs(bal) <= 1e-8 else EXIT_NUMERICAL
    ref = args.oracle or str(Path(path).with_suffix("")) + "_reference.csv"
    ref_name = Path(ref).name
    try:
        if Path(ref).exists():
            ids, mags, _ = dm.read_reference_voltages(ref)
        else:
            import tempfile
            with tempfile.NamedTemporaryFile("w", suffix=".csv", delete=False) as fh:
                fh.write(read_fixture(ref_name))
            ids, mags, _ = dm.read_reference_voltages(fh.name)
    except (FileNotFoundError, ValueError) as exc:
        raise CliInputError("reference", f"missing or bad reference fixture: {ref} ({exc})")
    res = dm.zbus_iterate(model)
    plan = engine.zbus_plan_for(model, 0)
    plan.set_network(model)
    sc = dm.base_distribution_scenario(model)
    kcl = float(plan.kirchhoff(res.v[None, :].copy(), np.ascontiguousarray(sc.wye_s[None, :]),
                               np.ascontiguousarray(sc.delta_s[None, :]))[0])
    pos = {k: i for i, k in enumerate(model.reduced_ids())}
    missing = [i for i in ids if i not in pos]
    if missing:
        raise CliInputError("reference", f"reference ids not in network: {missing[:5]}")
    dev = float(np.abs(np.array([abs(res.v[pos[i]]) for i in ids]) - mags).max())
    thr = args.tol if args.tol is not None else 1e-3
    print("quantity                     value")
    print(f"node-phases compared         {len(ids)}")
    print(f"max |dVmag| vs reference     {dev:.3e}  (threshold {thr:.1e})")
    print(f"Kirchhoff residual (device)  {kcl:.3e}  (threshold 1.0e-08)")
    print(f"solver converged             {res.converged}")
    return EXIT_OK if res.converged and dev < thr else EXIT_NUMERICAL


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="acpf-b200", description="Batched AC power flow on B200 GPUs.")
    sub = ap.add_subparsers(dest="command", required=True)
    for name, fn in (("solve", cmd_solve), ("bench", cmd_bench), ("verify", cmd_verify)):
        p = sub.add_parser(name)
        p.add_argument("--case", required=True)
        p.add_argument("--kind", choices=("tx", "dist"))
        p.add_argument("--batch", type=int, default=1)
        p.add_argument("--seed", type=int, default=0)
        p.add_argument("--spread", type=float, default=0.2)
        p.add_argument("--tol", type=float, default=None)
        p.add_argument("--workers", type=int, default=1, help="accepted; the GPU decides")
        p.add_argument("--out", default=None)
        p.add_argument("--format", choices=("json", "csv"), default="json")
        p.add_argument("--oracle", default=None)
        p.add_argument("--precond", choices=("fd", "none"), default="fd",
                       help="GMRES preconditioner for --step gmres (reference cli.py:322-327)")
        p.add_argument("--step", choices=("lu", "gmres"), default="lu",
                       help="Newton step: exact sparse LU (default) or the reference's GMRES")
        p.add_argument("-v", "--verbose", action="count", default=0)
        p.set_defaults(fn=fn)
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.fn(args)
    except CliInputError as exc:
        print(f"error: {exc.code}: {exc}", file=sys.stderr)
        return EXIT_INPUT
    except (nm.CaseParseError, dm.SchemaError) as exc:
        print(f"error: schema: {exc}", file=sys.stderr)
        return EXIT_INPUT
    except (ValueError, OSError) as exc:
        print(f"error: input: {exc}", file=sys.stderr)
        return EXIT_INPUT


if __name__ == "__main__":
    sys.exit(main())
