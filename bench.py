#!/usr/bin/env python
"""Benchmark: converged power flows/sec on B200 (GBnetwork NR headline, EULV Z-Bus secondary).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port P bench.py --gpus N ...

A *step* is one pass of the hot path over one batch of synthetic scenarios
(BASELINE.json configs[2] GBnetwork NR, configs[3] EULV Z-Bus; per-GPU batch
fixed, so scaling is weak). Scenarios come from the reference's own seeded
generator (Philox multipliers U[0.8, 1.2], batch.py:45-60) on the reference
fixtures. ``value`` is measured with inputs resident in HBM (CUDA events on
the solve stream, barrier + synchronize around the K timed steps, max over
ranks); ``e2e`` is the same metric through the C-ABI with pinned host
buffers, H2D of the inputs and D2H of voltages/flags inside the timed
region. Inputs exceed L2 (2.1 GB NR, 0.23 GB Z-Bus), so no explicit flush.

``--impl reference`` times the reference algorithm's CPU path (the pinned
oracle restatement, oracle/, GMRES-FD Newton / LU Z-Bus) on all host cores.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

NR_CASE, NR_SEED = "gb2224", 10010
ZB_CASE, ZB_SEED = "eulv", 10011
METRIC = "converged power flows/sec (GBnetwork NR, EULV Z-Bus) at 1/2/4/8 B200 vs CPU"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--nr-batch", type=int, default=65536, help="NR scenarios per GPU per step")
    ap.add_argument("--zb-batch", type=int, default=262144, help="Z-Bus scenarios per GPU per step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=64, help="scenarios per reference-arm step")
    ap.add_argument("--cpu-baseline-sample", type=int, default=1024,
                    help="scenarios of the cpu_baseline measurement on all host cores")
    ap.add_argument("--global-batch", type=int, default=0,
                    help="strong scaling: split this many scenarios over the ranks (BASELINE configs[4]: 1048576)")
    ap.add_argument("--sweep", action="store_true", help="batch-size sweeps of configs[2]/[3] (1 GPU)")
    ap.add_argument("--no-extra-configs", action="store_true")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md clocks line)
# ---------------------------------------------------------------------------


class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self) -> dict:
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)),
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------


def nr_setup(case: str):
    import paper_2605_14103_b200 as pf
    from paper_2605_14103_b200.fixtures import load_transmission

    net = load_transmission(case)
    model = pf.build_transmission_model(net)
    return model, pf.transmission_base(net, model.part)


def zb_setup(case: str):
    import paper_2605_14103_b200 as pf
    from paper_2605_14103_b200.fixtures import load_distribution

    model = pf.build_zbus_model(load_distribution(case))
    return model, pf.distribution_base(model)


def build_nr(rank, world, batch):
    """Host-side inputs (the CPU arm): rows rank*batch .. of the seeded batch."""
    import paper_2605_14103_b200 as pf

    model, base = nr_setup(NR_CASE)
    spec = pf.ScenarioSpec(count=batch * world, seed=NR_SEED)
    p, q = pf.make_scenario_arrays(base, spec, start=rank * batch, count=batch)
    return model, p, q


def build_zb(rank, world, batch):
    import paper_2605_14103_b200 as pf

    model, base = zb_setup(ZB_CASE)
    spec = pf.ScenarioSpec(count=batch * world, seed=ZB_SEED, target="distribution")
    sw, sd = pf.make_scenario_arrays(base, spec, start=rank * batch, count=batch)
    return model, sw, sd


def pinned_from(t):
    """Pinned host copy of a device tensor, as a numpy array."""
    import torch
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t)
    return h.numpy()


def pinned_outputs(outs: dict) -> dict:
    import torch
    res = {}
    for k, v in outs.items():
        t = torch.empty(v.shape, dtype=getattr(torch, str(v.dtype)), pin_memory=True)
        res[k] = t.numpy()
    return res


def time_device(fn, steps, warmup, stream, dev):
    """K timed steps bracketed by barrier + synchronize; CUDA events on `stream`."""
    import torch
    import torch.distributed as dist

    for _ in range(warmup):
        fn()
    torch.cuda.synchronize(dev)
    if dist.is_initialized():
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    if dist.is_initialized():
        dist.barrier()
    return e0.elapsed_time(e1) / 1e3


def time_host(fn, steps, warmup, dev):
    import torch
    import torch.distributed as dist

    for _ in range(warmup):
        fn()
    torch.cuda.synchronize(dev)
    if dist.is_initialized():
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        fn()
    torch.cuda.synchronize(dev)
    t = time.perf_counter() - t0
    if dist.is_initialized():
        dist.barrier()
    return t


def traffic_from_profiles(kernel: str, batch: int):
    """dram bytes per launch from a committed ncu --set full summary, if one
    matches this kernel and batch (profiles/ncu_traffic.json)."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    try:
        d = json.loads(p.read_text())
        e = d.get(kernel)
        if e and int(e.get("batch", -1)) == batch:
            return float(e["dram_bytes_per_launch"])
    except Exception:
        pass
    return None


PINNED_E2E_MAX_BYTES = 24 << 30  # host-pointer e2e needs the shard in pinned host memory


def nr_workload(args, dev, stream, local, case, seed, start, count, e2e=True, api=False, roof=True):
    """One NR step = one batched solve of rows start..start+count of the seeded
    batch, inputs generated on the device (bitwise the reference generator)."""
    import torch
    from paper_2605_14103_b200 import peaks, roofline, shard

    model, base = nr_setup(case)
    plan = model.plan(local)
    pt, qt = plan.scenarios(base, seed, start, count, 0.2, device=dev)
    out = plan.alloc_outputs(count, like=pt)
    acc = [0, 0.0]

    def step():  # enqueued, no host sync (device-pointer solves are stream-ordered)
        plan.solve(pt, qt, 1e-8, 20, out=out, stream=stream)

    with ClockSampler(local) as clk:
        for _ in range(args.warmup):
            step()
        t = time_device(step, args.steps, 0, stream, dev)
    ms, nl = plan.last_timing()  # the last solve's kernel time and launch count
    acc[:] = [nl * args.steps, ms * args.steps]
    t = shard.max_over_ranks(t, dev)
    conv = shard.sum_over_ranks(int(out["converged"].sum().item()), dev)
    its = out["iterations"].cpu().numpy()
    r = dict(value=conv * args.steps / t, t=t, launches=acc[0], clocks=clk.summary(),
             iterations=np.unique(its).tolist(), nnz_lu=plan.info["nnz_lu"], model=model)
    if roof:
        solve_s = acc[1] / 1e3 / args.steps
        nj = model.part.n_theta + model.part.n_q
        alg = float(roofline.nr_bytes_per_scenario(its, model.net.n, nj, plan.info["nnz_lu"]).sum())
        exe = float(roofline.nr_bytes_per_scenario_executed(its, model.net.n, nj, plan.info["nnz_lu"]).sum())
        hbm, hbm_src = peaks.hbm_gbs()
        traffic = traffic_from_profiles("nr_solve", count)
        r["roofline"] = {
            "bound": "hbm", "achieved": alg / solve_s / 1e9, "peak": hbm, "unit": "GB/s",
            "frac": alg / solve_s / 1e9 / hbm, "traffic": traffic,
            "kernel": "nr_factor_kernel (+ back/mismatch launches of one solve)",
            "algorithmic_bytes_per_launch": alg,
            # step 0 uses the flat-start LU shared by every scenario: the
            # pinned formula counts K factor passes, K-1 are executed
            "algorithmic_bytes_executed_per_launch": exe,
            "achieved_executed": exe / solve_s / 1e9, "frac_executed": exe / solve_s / 1e9 / hbm,
            "launch_unit": f"one batched Newton solve ({acc[0] // max(1, args.steps)} launches)",
            "avg_launch_ms": solve_s * 1e3, "peak_source": hbm_src,
            # measured DRAM bytes of the same launch sequence / its device time
            "traffic_GBps": traffic / solve_s / 1e9 if traffic else None,
            "traffic_frac": traffic / solve_s / 1e9 / hbm if traffic else None}
    if e2e:
        inb = (pt.numel() + qt.numel()) * 8
        outb = sum(v.numel() * v.element_size() for v in out.values())
        if inb + outb <= PINNED_E2E_MAX_BYTES:
            hp, hq = pinned_from(pt), pinned_from(qt)
            hout = pinned_outputs(plan.alloc_outputs(count))
            te = time_host(lambda: plan.solve(hp, hq, 1e-8, 20, out=hout), args.steps, 1, dev)
            te = shard.max_over_ranks(te, dev)
            ce = shard.sum_over_ranks(int(hout["converged"].sum()), dev)
            r["e2e"] = {"value": ce * args.steps / te, "unit": "converged flows/s",
                        "h2d_bytes_per_step": int(hp.nbytes + hq.nbytes) * shard.dist_env()[2],
                        "d2h_bytes_per_step": int(sum(v.nbytes for v in hout.values())) * shard.dist_env()[2]}
            if api:
                r["api"] = nr_api(args, model, hp, hq, dev)
            del hp, hq, hout
        else:
            r["e2e"] = None
    del pt, qt, out
    torch.cuda.empty_cache()
    return r


def nr_api(args, model, hp, hq, dev):
    """The drop-in Python API a user calls: transmission.batch_newton_solve on
    the scenario list make_scenarios returns (array-backed, page-locked tables,
    results.TransmissionScenarios), results returned as NewtonResult records
    backed by solver-allocated page-locked arrays (results.NewtonResults)."""
    import paper_2605_14103_b200 as pf
    from paper_2605_14103_b200 import shard
    from paper_2605_14103_b200.results import TransmissionScenarios

    scen = TransmissionScenarios(hp, hq)
    box = {}

    def step():
        box["r"] = pf.batch_newton_solve(model, scen)

    # two untimed calls: the pinned result buffers of two consecutive calls are
    # alive at once (the previous results until the new ones replace them)
    t = time_host(step, args.steps, 2, dev)
    t = shard.max_over_ranks(t, dev)
    conv = shard.sum_over_ranks(int(box["r"].converged().sum()), dev)
    return {"value": conv * args.steps / t, "unit": "converged flows/s",
            "call": "batch_newton_solve(model, make_scenarios-style TransmissionScenarios) -> NewtonResults",
            "host_memory": "page-locked scenario tables in (as make_scenarios builds them), "
                           "solver-allocated page-locked result tables out"}


def zb_api(args, model, hsw, hsd, dev):
    """distribution.batch_zbus_solve on the array-backed scenario list
    make_scenarios returns, results as FixedPointResult records over
    page-locked tables (results.ZbusResults)."""
    import paper_2605_14103_b200 as pf
    from paper_2605_14103_b200 import shard
    from paper_2605_14103_b200.results import DistributionScenarios

    scen = DistributionScenarios(hsw, hsd)
    box = {}

    def step():
        box["r"] = pf.batch_zbus_solve(model, scen)

    t = time_host(step, args.steps, 2, dev)
    t = shard.max_over_ranks(t, dev)
    conv = shard.sum_over_ranks(int(box["r"].converged().sum()), dev)
    return {"value": conv * args.steps / t, "unit": "converged flows/s",
            "call": "batch_zbus_solve(model, make_scenarios-style DistributionScenarios) -> ZbusResults",
            "host_memory": "page-locked scenario tables in, solver-allocated page-locked result tables out"}


def zb_workload(args, dev, stream, local, case, seed, start, count, e2e=True, roof=True, api=False):
    import torch
    from paper_2605_14103_b200 import engine, peaks, roofline, shard

    zmodel, base = zb_setup(case)
    zplan = engine.zbus_plan_for(zmodel, local)
    swt, sdt = zplan.scenarios(base, seed, start, count, 0.2, device=dev)
    sdt = sdt.reshape(count, -1).contiguous()
    zout = zplan.alloc_outputs(count, like=swt)
    acc = [0, 0.0]

    def step():  # enqueued, no host sync
        zplan.solve(swt, sdt, 1e-9, 100, out=zout, stream=stream)

    with ClockSampler(local) as clk:
        for _ in range(args.warmup):
            step()
        tz = time_device(step, args.steps, 0, stream, dev)
    ms, nl = zplan.last_timing()
    acc[:] = [nl * args.steps, ms * args.steps]
    tz = shard.max_over_ranks(tz, dev)
    zconv = shard.sum_over_ranks(int(zout["converged"].sum().item()), dev)
    zits = zout["iterations"].cpu().numpy()
    r = dict(value=zconv * args.steps / tz, t=tz, launches=acc[0], clocks=clk.summary(),
             iterations=np.unique(zits).tolist())
    if roof:
        nloads = zmodel.wye_idx.size + zmodel.delta_p.size
        zk = acc[1] / 1e3 / max(1, acc[0])
        zper = count / max(1, acc[0] / args.steps)
        zflops = float(roofline.zbus_flops_per_scenario(zits, zmodel.n, zmodel.load_cols.size,
                                                        nloads).mean()) * zper
        # the kernel forms each complex product with 3 real DMMA products
        # (zbus_kernel.cu): the tensor pipe executes 6 of the 8 algorithmic flops
        zexec = float(((zits.astype(np.float64) + 1) * 6.0 * zmodel.n * zmodel.load_cols.size).mean()) * zper
        fp, fp_src = peaks.fp64_tflops()
        r["roofline"] = {"bound": "tensor", "achieved": zflops / zk / 1e12, "peak": fp, "unit": "TFLOP/s",
                         "frac": zflops / zk / 1e12 / fp,
                         "traffic": traffic_from_profiles("zbus_kernel", count),
                         "kernel": "zbus_kernel<32> (16 warps)", "algorithmic_flops_per_launch": zflops,
                         "avg_launch_ms": zk * 1e3, "peak_source": fp_src,
                         "complex_product": "3-multiply (Zr(Ir+Ii), (Zr+Zi)Ii, (Zi-Zr)Ir)",
                         "dmma_executed_tflops": zexec / zk / 1e12, "dmma_executed_frac": zexec / zk / 1e12 / fp}
    if e2e:
        inb = (swt.numel() + sdt.numel()) * 16
        outb = sum(v.numel() * v.element_size() for v in zout.values())
        if inb + outb <= PINNED_E2E_MAX_BYTES:
            hsw, hsd = pinned_from(swt), pinned_from(sdt)
            hz = pinned_outputs(zplan.alloc_outputs(count))
            tze = time_host(lambda: zplan.solve(hsw, hsd, 1e-9, 100, out=hz), args.steps, 1, dev)
            tze = shard.max_over_ranks(tze, dev)
            ce = shard.sum_over_ranks(int(hz["converged"].sum()), dev)
            r["e2e"] = {"value": ce * args.steps / tze, "unit": "converged flows/s",
                        "h2d_bytes_per_step": int(hsw.nbytes + hsd.nbytes) * shard.dist_env()[2],
                        "d2h_bytes_per_step": int(sum(v.nbytes for v in hz.values())) * shard.dist_env()[2]}
            if api:
                r["api"] = zb_api(args, zmodel, hsw, hsd, dev)
            del hsw, hsd, hz
        else:
            r["e2e"] = None
    del swt, sdt, zout
    torch.cuda.empty_cache()
    return r


def run_ours(args, rank, local, world):
    """Headline NR (configs[2]) + secondary Z-Bus (configs[3]) per GPU; with
    --global-batch the batch (configs[4], 2^20) is split over the ranks
    (strong scaling), else every rank solves --nr-batch / --zb-batch rows of
    its own (weak scaling)."""
    import torch
    from paper_2605_14103_b200 import shard

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream(dev)
    if args.global_batch:
        a, b = shard.shard_range(args.global_batch, rank, world)
        nr_rows = zb_rows = (a, b - a)
    else:
        nr_rows = (rank * args.nr_batch, args.nr_batch)
        zb_rows = (rank * args.zb_batch, args.zb_batch)
    res = {"nr": nr_workload(args, dev, stream, local, NR_CASE, NR_SEED, *nr_rows, api=not args.global_batch),
           "zb": zb_workload(args, dev, stream, local, ZB_CASE, ZB_SEED, *zb_rows, api=not args.global_batch)}
    if not args.global_batch and not args.no_extra_configs:
        # BASELINE configs[0] (IEEE 14-bus NR x 1024) and configs[1] (IEEE13 Z-Bus x 4096)
        c1 = nr_workload(args, dev, stream, local, "case14", 1010, rank * 1024, 1024, roof=False)
        c2 = zb_workload(args, dev, stream, local, "ieee13", 5050, rank * 4096, 4096, roof=False)
        res["extra"] = {
            "configs[0] IEEE 14-bus NR x 1024/GPU (case14, seed 1010)": {
                "value": c1["value"], "ms_per_step": c1["t"] / args.steps * 1e3,
                "iterations": c1["iterations"], "e2e": c1["e2e"]},
            "configs[1] IEEE 13-node Z-Bus x 4096/GPU (ieee13, seed 5050)": {
                "value": c2["value"], "ms_per_step": c2["t"] / args.steps * 1e3,
                "iterations": c2["iterations"], "e2e": c2["e2e"]}}
    return res


def run_sweep(args):
    """BASELINE configs[2]/[3] batch sweeps on one GPU: device-resident and
    e2e throughput per batch size (one JSON line per point)."""
    import torch

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream(dev)
    for b in (1, 8, 64, 256, 1024, 4096, 16384, 65536):
        r = nr_workload(args, dev, stream, 0, NR_CASE, NR_SEED, 0, b, roof=b >= 1024)
        print(json.dumps({"sweep": "configs[2] GBnetwork NR", "batch": b, "value": r["value"],
                          "ms_per_step": r["t"] / args.steps * 1e3, "e2e": r["e2e"],
                          "launches_per_step": r["launches"] / args.steps, "iterations": r["iterations"],
                          "roofline_frac": r.get("roofline", {}).get("frac"), "clocks": r["clocks"]}), flush=True)
    for b in (1, 8, 64, 256, 1024, 4096, 16384, 65536, 262144):
        r = zb_workload(args, dev, stream, 0, ZB_CASE, ZB_SEED, 0, b, roof=b >= 1024)
        print(json.dumps({"sweep": "configs[3] EULV Z-Bus", "batch": b, "value": r["value"],
                          "ms_per_step": r["t"] / args.steps * 1e3, "e2e": r["e2e"],
                          "iterations": r["iterations"], "roofline_frac": r.get("roofline", {}).get("frac"),
                          "clocks": r["clocks"]}), flush=True)
    return 0


# ---------------------------------------------------------------------------
# CPU path (reference algorithm restated in oracle/) -- baseline / reference arm
# ---------------------------------------------------------------------------

_CPU = {}


def _cpu_init(kind):
    import paper_2605_14103_b200 as pf
    from oracle import nr as onr
    from oracle import zbus as ozb
    if kind == "nr":
        model, p, q = build_nr(0, 1, 1)
        st = pf.flat_start(model.net, model.part)
        case = onr.NrCase(model.y.csr, model.part.theta_block, model.part.q_block, st.theta, st.vmag)
        case.fd()
        _CPU["nr"] = (case, model)
    else:
        model = pf.build_zbus_model(__import__("paper_2605_14103_b200.fixtures", fromlist=["x"]).load_distribution(ZB_CASE))
        _CPU["zb"] = (ozb.ZbCase(model.y_nn, model.v0, model.wye_idx, model.delta_p, model.delta_q,
                                 model.voltage_floor), model)


def _cpu_nr(args):
    from oracle import nr as onr
    p, q = args
    return onr.newton(_CPU["nr"][0], p, q).converged


def _cpu_zb(args):
    from oracle import zbus as ozb
    sw, sd = args
    return ozb.zbus(_CPU["zb"][0], sw, sd).converged


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_throughput(kind: str, count: int, steps: int, warmup: int, workers: int = 0):
    """Reference CPU algorithm over `workers` host cores (0 = all; fork pool,
    BLAS pinned to one thread per worker, as the reference's run_batch does,
    batch.py:280-344, _threads.py:18-23)."""
    import multiprocessing as mp
    from threadpoolctl import threadpool_limits
    import paper_2605_14103_b200 as pf

    cores = workers or os.cpu_count() or 1
    if kind == "nr":
        model, _, _ = build_nr(0, 1, 1)
        base = pf.transmission_base(model.net, model.part)
        p, q = pf.make_scenario_arrays(base, pf.ScenarioSpec(count=count, seed=NR_SEED))
        work = list(zip(p, q))
        fn = _cpu_nr
    else:
        zm, sw, sd = build_zb(0, 1, count)
        work = list(zip(sw, sd))
        fn = _cpu_zb
    _cpu_init(kind)
    ctx = mp.get_context("fork")
    with threadpool_limits(limits=1):
        with ctx.Pool(cores) as pool:
            for _ in range(warmup):
                pool.map(fn, work[:cores], chunksize=1)
            t0 = time.perf_counter()
            nconv = 0
            for _ in range(steps):
                nconv += sum(pool.map(fn, work, chunksize=max(1, len(work) // (cores * 4))))
            t = time.perf_counter() - t0
    return nconv / t, cores, t


def cpu_baselines(sample: int) -> tuple:
    """cpu_baseline objects (NR, Z-Bus): all host cores over `sample`
    scenarios, plus one core over a 32-scenario sample."""
    model = cpu_model()
    out = []
    for kind, case, seed, alg in (("nr", NR_CASE, NR_SEED, "oracle GMRES-FD Newton (reference algorithm)"),
                                  ("zb", ZB_CASE, ZB_SEED, "oracle LU Z-Bus (reference algorithm)")):
        v, cores, t = cpu_throughput(kind, sample, 1, 1)
        v1, _, t1 = cpu_throughput(kind, 32, 1, 1, workers=1)
        out.append({"value": v, "unit": "converged flows/s", "cores": cores, "kind": "port",
                    "sample": f"{sample} {case} scenarios (seed {seed}), {alg}, fork pool of {cores} "
                              f"({t:.1f} s)",
                    "cpu_model": model, "single_core": {"value": v1, "cores": 1,
                                                        "sample": f"32 {case} scenarios ({t1:.1f} s)"}})
    return tuple(out)


# ---------------------------------------------------------------------------


def main():
    args = parse()
    rank, local, world = int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), \
        int(os.environ.get("WORLD_SIZE", 1))
    if args.impl == "reference":
        if rank != 0:
            return 0
        steps = max(1, args.steps)
        v, cores, t = cpu_throughput("nr", args.cpu_sample, steps, 1)
        zv, zcores, zt = cpu_throughput("zb", args.cpu_sample, steps, 1)
        line = {
            "metric": METRIC, "value": v, "unit": "converged flows/s", "n_gpus": args.gpus,
            "steps": steps, "warmup": args.warmup, "ms_per_step": t / steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: seeded Philox load multipliers U[0.8,1.2] (reference generator)",
            "impl": "reference",
            "config": {"workload": f"GBnetwork ({NR_CASE}) Newton-Raphson, CPU sample of "
                                   f"{args.cpu_sample} scenarios per step", "seed": NR_SEED},
            "cpu_baseline": {"value": v, "unit": "converged flows/s", "cores": cores, "kind": "port",
                             "sample": f"{args.cpu_sample} {NR_CASE} scenarios x {steps} steps, "
                                       f"oracle GMRES-FD Newton, fork pool of {cores}",
                             "cpu_model": cpu_model()},
            "e2e": {"value": v, "unit": "converged flows/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "secondary": {"workload": f"EULV ({ZB_CASE}) Z-Bus", "value": zv,
                          "unit": "converged flows/s", "cores": zcores,
                          "sample": f"{args.cpu_sample} scenarios x {steps} steps"},
        }
        print(json.dumps(line), flush=True)
        return 0

    import torch
    import torch.distributed as dist

    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if args.sweep:
        return run_sweep(args)
    res = run_ours(args, rank, local, world)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baselines(args.cpu_baseline_sample)
    if rank == 0:
        nr, zb = res["nr"], res["zb"]
        strong = bool(args.global_batch)
        nr_b = args.global_batch if strong else args.nr_batch * world
        zb_b = args.global_batch if strong else args.zb_batch * world
        line = {
            "metric": METRIC, "value": nr["value"], "unit": "converged flows/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": nr["t"] / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: seeded Philox load multipliers U[0.8,1.2] on the reference "
                    "fixtures (reference generator, batch.py:45-60; rows generated on the GPU, bitwise)",
            "config": {"workload": (f"GBnetwork ({NR_CASE}, 2224 buses) Newton-Raphson, {nr_b} scenarios "
                                    f"split over {world} GPU(s) (BASELINE configs[4])") if strong else
                                   (f"GBnetwork ({NR_CASE}, 2224 buses) Newton-Raphson, "
                                    f"{args.nr_batch} scenarios/GPU/step (BASELINE configs[2])"),
                       "batch_per_gpu": nr_b // world, "global_batch": nr_b,
                       "seed": NR_SEED, "parallelism": f"scenario shards x{world}, no collective",
                       "l2": "inputs (2.1 GB/GPU) larger than L2; no flush",
                       "nnz_lu": nr["nnz_lu"], "newton_iterations": nr["iterations"]},
            "roofline": nr["roofline"],
            "cpu_baseline": cpu[0] if cpu else None,
            "e2e": nr["e2e"],
            "gpu_launches": nr["launches"] + 0,
            "clocks": nr["clocks"],
            "secondary": {
                "workload": (f"EULV ({ZB_CASE}, 2724 phases) Z-Bus, {zb_b} scenarios split over {world} "
                             "GPU(s) (BASELINE configs[4])") if strong else
                            (f"EULV ({ZB_CASE}, 2724 phases) Z-Bus, {args.zb_batch} scenarios/GPU/step "
                             "(BASELINE configs[3])"),
                "value": zb["value"], "unit": "converged flows/s",
                "ms_per_step": zb["t"] / args.steps * 1e3, "roofline": zb["roofline"],
                "e2e": zb["e2e"], "api": zb.get("api"), "gpu_launches": zb["launches"], "clocks": zb["clocks"],
                "iterations": zb["iterations"], "cpu_baseline": cpu[1] if cpu else None},
        }
        if nr.get("api"):
            line["api"] = nr["api"]
        if res.get("extra"):
            line["extra_configs"] = res["extra"]
        if strong and nr["e2e"] is None:
            line["e2e_note"] = ("shard larger than the pinned host staging bound "
                                f"({PINNED_E2E_MAX_BYTES >> 30} GiB); see the weak-scaling line's e2e")
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
