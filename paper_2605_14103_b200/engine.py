"""ctypes binding of libacpf.so (include/acpf.h) and the device plans.

This is the only bridge between the host API (reference-shaped dataclasses)
and the CUDA engine. There is no CPU fallback: if the library or a GPU is
missing every solve raises :class:`EngineUnavailable`.

Batch buffers may be numpy arrays (host pointers, ``ACPF_HOST_PTRS``: the
library stages through device memory) or CUDA ``torch`` tensors
(``ACPF_DEVICE_PTRS``); torch is used for device memory only.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from pathlib import Path

import numpy as np

_LIB_PATH = Path(__file__).resolve().parent / "libacpf.so"

ACPF_HOST_PTRS = 0
ACPF_DEVICE_PTRS = 1

NR_CONVERGED, NR_MAX_ITER, NR_NONFINITE, NR_VMAG_LE0, NR_ZERO_PIVOT = range(5)
ZB_CONVERGED, ZB_MAX_ITER, ZB_FLOOR = range(3)

EXPORTED = (
    "acpf_last_error", "acpf_abi_version", "acpf_device_count",
    "acpf_nr_plan_create", "acpf_solve_result_json", "acpf_report_csv", "acpf_ybus_build", "acpf_y3_build", "acpf_nr_ordering", "acpf_nr_analyze", "acpf_nr_flat_start_solve", "acpf_nr_plan_info_get",
    "acpf_nr_plan_structure",
    "acpf_nr_solve", "acpf_nr_solve_start", "acpf_nr_last_timing", "acpf_nr_plan_destroy",
    "acpf_zbus_plan_create", "acpf_zbus_solve", "acpf_zbus_last_timing",
    "acpf_zbus_plan_destroy", "acpf_philox_multipliers", "acpf_nr_scenarios",
    "acpf_zbus_scenarios", "acpf_nr_plan_set_branches", "acpf_nr_certify",
    "acpf_zbus_plan_set_network", "acpf_zbus_kirchhoff", "acpf_zbus_reduce",
    "acpf_nr_plan_set_fd", "acpf_nr_solve_gmres",
)


class EngineUnavailable(RuntimeError):
    """libacpf.so missing/unbuildable or no CUDA device: there is no fallback."""


class EngineError(RuntimeError):
    """A C-ABI call returned a negative acpf_status."""


class NrPlanInfo(C.Structure):
    _fields_ = [
        ("n_bus", C.c_int32), ("n_theta", C.c_int32), ("n_q", C.c_int32), ("n_j", C.c_int32),
        ("nnz_y", C.c_int32), ("nnz_j", C.c_int32), ("nnz_lu", C.c_int64), ("n_pairs", C.c_int64),
        ("group", C.c_int32), ("etree_height", C.c_int32),
        ("workspace_bytes_per_group", C.c_int64),
    ]


_lib = None

P = C.c_void_p
I32 = C.c_int32
I64 = C.c_int64
U32 = C.c_uint32
D = C.c_double


def load_library(path: str | os.PathLike | None = None):
    """Load (building first if stale and nvcc is present) and type the C-ABI."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    override = os.environ.get("ACPF_LIB")  # an alternative build of the same C-ABI
    target = Path(path) if path else (Path(override) if override else _LIB_PATH)
    if path is None and not override:
        try:
            from . import _build
            if _build._stale() and Path(_build.NVCC).exists():
                _build.build()
        except Exception as exc:  # a stale-but-present library still loads
            if not target.exists():
                raise EngineUnavailable(f"cannot build {target}: {exc}") from exc
    if not target.exists():
        raise EngineUnavailable(f"{target} not built (run __graft_entry__.build())")
    lib = C.CDLL(str(target))
    sig = {
        "acpf_last_error": (C.c_char_p, []),
        "acpf_abi_version": (I32, []),
        "acpf_device_count": (I32, []),
        "acpf_nr_plan_create": (I32, [I32, I32, P, P, P, P, I32, P, I32, P, P, P, P, P]),
        "acpf_nr_ordering": (I32, [I32, P, P, I32, P, I32, P]),
        "acpf_solve_result_json": (I32, [P, I64, P, P, P, P, P, I32, P, P, P, I32, P, C.c_char_p, P, I64,
                                          P]),
        "acpf_report_csv": (I32, [I64, P, P, P, P, P, C.c_char_p, P, I64, P]),
        "acpf_ybus_build": (I32, [I32, I32, P, P, P, P, P, P, P, P, P, P, I64, P, P, P, P, P]),
        "acpf_y3_build": (I32, [I32, I32, P, P, P, I64, P, P, P, P, P]),
        "acpf_nr_analyze": (I32, [I32, P, P, I32, P, I32, P, P, P]),
        "acpf_nr_flat_start_solve": (I32, [I32, P, P, P, P, I32, P, I32, P, P, P, P, P, P]),
        "acpf_nr_plan_info_get": (I32, [P, P]),
        "acpf_nr_plan_structure": (I32, [P, P, P]),
        "acpf_nr_solve": (I32, [P, I64, P, P, D, I32, P, P, P, P, P, P, U32, P]),
        "acpf_nr_solve_start": (I32, [P, I64, P, P, P, P, D, I32, P, P, P, P, P, P, U32, P]),
        "acpf_nr_last_timing": (I32, [P, P, P]),
        "acpf_nr_plan_destroy": (I32, [P]),
        "acpf_zbus_plan_create": (I32, [I32, I32, I32, P, P, P, I32, P, I32, P, P, D, P]),
        "acpf_zbus_solve": (I32, [P, I64, P, P, D, I32, P, P, P, P, P, P, P, U32, P]),
        "acpf_zbus_last_timing": (I32, [P, P, P]),
        "acpf_zbus_plan_destroy": (I32, [P]),
        "acpf_philox_multipliers": (I32, [C.c_uint64, I64, I64, I32, D, P, U32, P]),
        "acpf_nr_scenarios": (I32, [P, C.c_uint64, I64, I64, D, I32, P, P, P, P, P, P, P, U32, P]),
        "acpf_zbus_scenarios": (I32, [P, C.c_uint64, I64, I64, D, I32, P, P, P, P, P, U32, P]),
        "acpf_nr_plan_set_branches": (I32, [P, I32, P, P, P, P]),
        "acpf_nr_certify": (I32, [P, I64, P, P, P, P, P, P, P, U32, P]),
        "acpf_zbus_plan_set_network": (I32, [P, P, P, P, P]),
        "acpf_zbus_kirchhoff": (I32, [P, I64, P, P, P, P, U32, P]),
        "acpf_zbus_reduce": (I32, [I32, I32, P, P, P, P, I32, P, P, P]),
        "acpf_nr_plan_set_fd": (I32, [P, P, P, P, P, P]),
        "acpf_nr_solve_gmres": (I32, [P, I64, P, P, D, I32, D, I32, I32, I32, P, P, P, P, P, P, P, P, P,
                                      P, U32, P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def _check(rc: int) -> None:
    if rc != 0:
        msg = _lib.acpf_last_error().decode(errors="replace") if _lib else ""
        raise EngineError(f"acpf status {rc}: {msg}")


def require_device(device: int = 0) -> None:
    lib = load_library()
    n = lib.acpf_device_count()
    if n <= device:
        raise EngineUnavailable(f"no CUDA device {device} (found {n}); the engine has no CPU path")


def _ptr(a) -> int | None:
    """Raw address of a numpy array or torch tensor (None -> NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if not a.flags.c_contiguous:
            raise ValueError("arrays passed to the engine must be C-contiguous")
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise ValueError("tensors passed to the engine must be contiguous")
        return a.data_ptr()
    raise TypeError(f"unsupported buffer type {type(a)!r}")


def _is_device(a) -> bool:
    return hasattr(a, "is_cuda") and bool(a.is_cuda)


def _stream_ptr(stream, like=None) -> int | None:
    """cudaStream_t for a call; device tensors default to torch's current
    stream (device-pointer solves are stream-ordered and asynchronous)."""
    if stream is None:
        if like is not None and _is_device(like):
            import torch
            return int(torch.cuda.current_stream(like.device).cuda_stream) or None
        return None
    return int(getattr(stream, "cuda_stream", stream))


class ResultMeta(C.Structure):
    _fields_ = [("case_name", C.c_char_p), ("kind", C.c_char_p), ("seed", C.c_int64), ("spread", C.c_double),
                ("batch", C.c_int64), ("worker_count", C.c_int64), ("total_wall_time", C.c_double),
                ("throughput", C.c_double)]


def _report_arrays(converged, iterations, residual, wall_time, errors):
    n = len(converged)
    conv = np.ascontiguousarray(converged, dtype=np.uint8)
    its = np.ascontiguousarray(iterations, dtype=np.int32)
    res = np.ascontiguousarray(residual, dtype=np.float64)
    wall = np.ascontiguousarray(np.broadcast_to(np.asarray(wall_time, dtype=np.float64), (n,)))
    errs = None
    keep = []
    if errors is not None and any(e is not None for e in errors):
        errs = (C.c_char_p * n)()
        for k, e in enumerate(errors):
            if e is not None:
                b = str(e).encode("utf-8", "surrogatepass")
                keep.append(b)
                errs[k] = b
    return n, conv, its, res, wall, errs, keep


def _text_out(call, path):
    """path -> written file (returns None); no path -> the text, sized first."""
    if path is not None:
        _check(call(str(path).encode(), None, 0, None))
        return None
    n = C.c_int64(0)
    _check(call(None, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    _check(call(None, buf, n.value, C.byref(n)))
    return buf.raw[:n.value].decode("utf-8")


def solve_result_json(meta: dict, converged, iterations, residual, wall_time, errors=None, state_a=None,
                      state_b=None, has_solution=None, node_phase_ids=None, path=None):
    """acpflow-solve-result/1 document written natively (acpf_solve_result_json):
    byte-identical to json.dumps(doc, indent=1) + "\n" of the reference's
    `solve` (cli.py:141-180). state_a/state_b: [count][n] theta/vmag (tx) or
    v_re/v_im (dist)."""
    lib = load_library()
    n, conv, its, res, wall, errs, keep = _report_arrays(converged, iterations, residual, wall_time, errors)
    m = ResultMeta(str(meta["case"]).encode(), str(meta["kind"]).encode(), int(meta["seed"]),
                   float(meta["spread"]), int(meta["batch"]), int(meta.get("worker_count", 1)),
                   float(meta["total_wall_time"]), float(meta["throughput"]))
    a = None if state_a is None else np.ascontiguousarray(state_a, dtype=np.float64)
    b = None if state_b is None else np.ascontiguousarray(state_b, dtype=np.float64)
    ns = 0 if a is None else (a.shape[1] if a.ndim == 2 else 0)
    has = None if has_solution is None else np.ascontiguousarray(has_solution, dtype=np.uint8)
    ids = None
    if node_phase_ids is not None:
        enc = [str(x).encode("utf-8") for x in node_phase_ids]
        keep.extend(enc)
        ids = (C.c_char_p * max(len(enc), 1))(*enc)
    n_ids = 0 if node_phase_ids is None else len(node_phase_ids)
    return _text_out(lambda pth, out, cap, ln: lib.acpf_solve_result_json(
        C.byref(m), n, _ptr(conv), _ptr(its), _ptr(res), _ptr(wall), errs, ns, _ptr(a), _ptr(b), _ptr(has),
        n_ids, ids, pth, out, cap, ln), path)


def report_csv(converged, iterations, residual, wall_time, errors=None, path=None):
    """report_to_csv written natively (acpf_report_csv), byte-identical to the
    reference's batch.py:379-387."""
    lib = load_library()
    n, conv, its, res, wall, errs, keep = _report_arrays(converged, iterations, residual, wall_time, errors)
    return _text_out(lambda pth, out, cap, ln: lib.acpf_report_csv(
        n, _ptr(conv), _ptr(its), _ptr(res), _ptr(wall), errs, pth, out, cap, ln), path)


def _csr_two_pass(call, n: int):
    """Run a host-only CSR builder twice: size query, then fill."""
    import scipy.sparse as sp
    nnz = C.c_int64(0)
    _check(call(0, None, None, None, None, C.byref(nnz)))
    k = nnz.value
    rp = np.empty(n + 1, dtype=np.int32)
    col = np.empty(max(k, 1), dtype=np.int32)
    re = np.empty(max(k, 1), dtype=np.float64)
    im = np.empty(max(k, 1), dtype=np.float64)
    _check(call(k, _ptr(rp), _ptr(col), _ptr(re), _ptr(im), C.byref(nnz)))
    val = np.empty(k, dtype=np.complex128)
    val.real, val.imag = re[:k], im[:k]
    y = sp.csr_matrix((val, col[:k].copy(), rp), shape=(n, n))
    y.has_sorted_indices = True
    return y


def ybus_build(n_bus: int, f, t, r, x, b_ch, tap, shift, in_service, gs, bs):
    """Native pi-model Ybus (acpf_ybus_build, host only) -> complex CSR."""
    lib = load_library()
    a32 = lambda v: np.ascontiguousarray(v, dtype=np.int32)  # noqa: E731
    f64 = lambda v: np.ascontiguousarray(v, dtype=np.float64)  # noqa: E731
    f, t = a32(f), a32(t)
    r, x, b_ch, tap, shift, gs, bs = map(f64, (r, x, b_ch, tap, shift, gs, bs))
    on = np.ascontiguousarray(in_service, dtype=np.uint8)
    return _csr_two_pass(lambda cap, rp, col, re, im, nz: lib.acpf_ybus_build(
        n_bus, f.size, _ptr(f), _ptr(t), _ptr(r), _ptr(x), _ptr(b_ch), _ptr(tap), _ptr(shift), _ptr(on),
        _ptr(gs), _ptr(bs), cap, rp, col, re, im, nz), n_bus)


def y3_build(n: int, blocks):
    """Native three-phase node-phase Y (acpf_y3_build, host only) from
    (block k x k complex, row node-phases, column node-phases) in stamp order."""
    lib = load_library()
    blocks = list(blocks)
    sizes = [len(r) for _, r, _ in blocks]
    ptr = np.zeros(len(blocks) + 1, dtype=np.int32)
    ptr[1:] = np.cumsum(sizes)
    idx = np.ascontiguousarray(np.concatenate([np.concatenate([r, c]) for _, r, c in blocks])
                               if blocks else np.zeros(0), dtype=np.int32)
    val = np.ascontiguousarray(np.concatenate([np.asarray(b, dtype=np.complex128).ravel() for b, _, _ in blocks])
                               if blocks else np.zeros(0, dtype=np.complex128)).view(np.float64)
    return _csr_two_pass(lambda cap, rp, col, re, im, nz: lib.acpf_y3_build(
        n, len(blocks), _ptr(ptr), _ptr(idx) if idx.size else None, _ptr(val) if val.size else None,
        cap, rp, col, re, im, nz), n)


ORDER_MIN_DEGREE, ORDER_MIN_FILL = 1, 2  # include/acpf.h ACPF_ORDER_*


def nr_ordering(y_csr, theta_block, kind: int = ORDER_MIN_FILL) -> np.ndarray:
    """Native fill-reducing elimination order of the 2x2 bus blocks
    (acpf_nr_ordering, host only): perm[k] = theta-block index of the bus
    eliminated k-th."""
    lib = load_library()
    y = y_csr.tocsr()
    y.sort_indices()
    rowptr = np.ascontiguousarray(y.indptr, dtype=np.int32)
    col = np.ascontiguousarray(y.indices, dtype=np.int32)
    tb = np.ascontiguousarray(theta_block, dtype=np.int32)
    out = np.empty(tb.size, dtype=np.int32)
    _check(lib.acpf_nr_ordering(y.shape[0], _ptr(rowptr), _ptr(col), tb.size, _ptr(tb), int(kind), _ptr(out)))
    return out


def nr_analyze(y_csr, theta_block, q_block, perm=None) -> dict:
    """Host-only symbolic analysis (no GPU): structure sizes for a network."""
    lib = load_library()
    y = y_csr.tocsr()
    y.sort_indices()
    rowptr = np.ascontiguousarray(y.indptr, dtype=np.int32)
    col = np.ascontiguousarray(y.indices, dtype=np.int32)
    tb = np.ascontiguousarray(theta_block, dtype=np.int32)
    qb = np.ascontiguousarray(q_block, dtype=np.int32)
    pm = None if perm is None else np.ascontiguousarray(perm, dtype=np.int32)
    info = NrPlanInfo()
    _check(lib.acpf_nr_analyze(y.shape[0], _ptr(rowptr), _ptr(col), tb.size, _ptr(tb), qb.size,
                               _ptr(qb), _ptr(pm), C.byref(info)))
    return {f: getattr(info, f) for f, _ in NrPlanInfo._fields_}


def nr_flat_start_solve(y_csr, theta_block, q_block, theta_init, vmag_init, rhs, perm=None):
    """Host-only: x = J(x0)^-1 rhs with the flat-start LU shared by every
    scenario's first Newton step (acpf_nr_flat_start_solve)."""
    lib = load_library()
    y = y_csr.tocsr()
    y.sort_indices()
    rowptr = np.ascontiguousarray(y.indptr, dtype=np.int32)
    col = np.ascontiguousarray(y.indices, dtype=np.int32)
    yr = np.ascontiguousarray(y.data.real, dtype=np.float64)
    yi = np.ascontiguousarray(y.data.imag, dtype=np.float64)
    tb = np.ascontiguousarray(theta_block, dtype=np.int32)
    qb = np.ascontiguousarray(q_block, dtype=np.int32)
    th = np.ascontiguousarray(theta_init, dtype=np.float64)
    vm = np.ascontiguousarray(vmag_init, dtype=np.float64)
    b = np.ascontiguousarray(rhs, dtype=np.float64)
    x = np.empty_like(b)
    pm = None if perm is None else np.ascontiguousarray(perm, dtype=np.int32)
    _check(lib.acpf_nr_flat_start_solve(y.shape[0], _ptr(rowptr), _ptr(col), _ptr(yr), _ptr(yi), tb.size,
                                        _ptr(tb), qb.size, _ptr(qb) if qb.size else None, _ptr(th), _ptr(vm),
                                        _ptr(pm), _ptr(b), _ptr(x)))
    return x


def _out_array(shape, dtype, device):
    if device is None:
        return np.empty(shape, dtype=dtype)
    import torch
    tdt = {np.float64: torch.float64, np.complex128: torch.complex128}[dtype]
    return torch.empty(shape, dtype=tdt, device=device)


def philox_multipliers(seed: int, start: int, count: int, n_elem: int, spread: float = 0.2,
                       device=None):
    """Rows start..start+count of generate_load_multipliers on the GPU
    (bitwise numpy's Philox4x64-10 stream keyed (seed, i))."""
    load_library()
    out = _out_array((count, n_elem), np.float64, device)
    flags = ACPF_DEVICE_PTRS if device is not None else ACPF_HOST_PTRS
    _check(_lib.acpf_philox_multipliers(int(seed), int(start), int(count), int(n_elem), float(spread),
                                        _ptr(out), flags, None))
    return out


# ---------------------------------------------------------------------------
# Newton plans
# ---------------------------------------------------------------------------


def branch_admittances(net):
    """In-service branches of a TransmissionNetwork as (from, to, y4, bus_gs):
    y4[k] = (yff, yft, ytf, ytt) of the pi model exactly as branch_flows
    forms them (reference transmission.py:453-481)."""
    idx = net.bus_index()
    f, t, y4 = [], [], []
    for br in net.branches:
        if not br.status:
            continue
        ys = 1.0 / complex(br.r, br.x)
        half_b = 0.5j * br.b_ch
        ratio = br.tap * np.exp(1j * br.shift)
        f.append(idx[br.from_bus])
        t.append(idx[br.to_bus])
        y4.append(((ys + half_b) / (br.tap * br.tap), -ys / np.conj(ratio), -ys / ratio, ys + half_b))
    gs = np.ascontiguousarray([b.gs for b in net.buses], dtype=np.float64)
    return (np.ascontiguousarray(f, dtype=np.int32), np.ascontiguousarray(t, dtype=np.int32),
            np.ascontiguousarray(np.array(y4, dtype=np.complex128).reshape(-1, 4)), gs)


class NrPlan:
    """Device plan for one transmission network (acpf_nr_plan_create)."""

    def __init__(self, y_csr, theta_block, q_block, theta_init, vmag_init, device: int = 0,
                 perm=None):
        require_device(device)
        lib = load_library()
        y = y_csr.tocsr()
        y.sort_indices()
        self.n_bus = y.shape[0]
        rowptr = np.ascontiguousarray(y.indptr, dtype=np.int32)
        col = np.ascontiguousarray(y.indices, dtype=np.int32)
        yre = np.ascontiguousarray(y.data.real, dtype=np.float64)
        yim = np.ascontiguousarray(y.data.imag, dtype=np.float64)
        tb = np.ascontiguousarray(theta_block, dtype=np.int32)
        qb = np.ascontiguousarray(q_block, dtype=np.int32)
        th0 = np.ascontiguousarray(theta_init, dtype=np.float64)
        vm0 = np.ascontiguousarray(vmag_init, dtype=np.float64)
        pm = None if perm is None else np.ascontiguousarray(perm, dtype=np.int32)
        h = P()
        _check(lib.acpf_nr_plan_create(device, self.n_bus, _ptr(rowptr), _ptr(col), _ptr(yre),
                                       _ptr(yim), tb.size, _ptr(tb), qb.size, _ptr(qb), _ptr(th0),
                                       _ptr(vm0), _ptr(pm), C.byref(h)))
        self._h = h
        self.device = device
        self.n_theta, self.n_q = int(tb.size), int(qb.size)
        info = NrPlanInfo()
        _check(lib.acpf_nr_plan_info_get(h, C.byref(info)))
        self.info = {f: getattr(info, f) for f, _ in NrPlanInfo._fields_}

    def structure(self):
        perm = np.empty(self.info["n_j"], dtype=np.int32)
        rp = np.empty(self.info["n_j"] + 1, dtype=np.int64)
        _check(_lib.acpf_nr_plan_structure(self._h, _ptr(perm), _ptr(rp)))
        return perm, rp

    def solve(self, p_spec, q_spec, tol: float, max_newton: int, out: dict | None = None,
              stream=None, theta_start=None, vmag_start=None) -> dict:
        """Solve a stacked batch. numpy in -> numpy out (host staging inside
        the library); CUDA tensors in -> CUDA tensors out (device pointers).
        ``theta_start``/``vmag_start`` ([batch][n_bus]): start state per
        scenario instead of the flat start (acpf_nr_solve_start)."""
        dev = _is_device(p_spec)
        b = int(p_spec.shape[0])
        if out is None:
            out = self.alloc_outputs(b, like=p_spec if dev else None)
        flags = ACPF_DEVICE_PTRS if dev else ACPF_HOST_PTRS
        outs = (_ptr(out["theta"]), _ptr(out["vmag"]), _ptr(out["converged"]), _ptr(out["iterations"]),
                _ptr(out["final_mismatch_inf"]), _ptr(out["status"]))
        if theta_start is None:
            _check(_lib.acpf_nr_solve(self._h, b, _ptr(p_spec), _ptr(q_spec), float(tol), int(max_newton),
                                      *outs, flags, _stream_ptr(stream, p_spec)))
        else:
            _check(_lib.acpf_nr_solve_start(self._h, b, _ptr(p_spec), _ptr(q_spec), _ptr(theta_start),
                                            _ptr(vmag_start), float(tol), int(max_newton), *outs, flags,
                                            _stream_ptr(stream, p_spec)))
        return out

    def alloc_outputs(self, b: int, like=None) -> dict:
        if like is not None:
            import torch
            kw = dict(device=like.device)
            return {
                "theta": torch.empty((b, self.n_bus), dtype=torch.float64, **kw),
                "vmag": torch.empty((b, self.n_bus), dtype=torch.float64, **kw),
                "converged": torch.empty(b, dtype=torch.uint8, **kw),
                "iterations": torch.empty(b, dtype=torch.int32, **kw),
                "final_mismatch_inf": torch.empty(b, dtype=torch.float64, **kw),
                "status": torch.empty(b, dtype=torch.int32, **kw),
            }
        from . import hostmem
        return {
            "theta": hostmem.empty((b, self.n_bus)), "vmag": hostmem.empty((b, self.n_bus)),
            "converged": hostmem.empty(b, np.uint8), "iterations": hostmem.empty(b, np.int32),
            "final_mismatch_inf": hostmem.empty(b), "status": hostmem.empty(b, np.int32),
        }

    def last_timing(self) -> tuple:
        ms, n = D(), I32()
        _check(_lib.acpf_nr_last_timing(self._h, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def scenarios(self, base, seed: int, start: int, count: int, spread: float = 0.2, device=None):
        """Seeded (p_spec, q_spec) rows generated on the GPU, bitwise
        batch.make_scenario_arrays(base, ScenarioSpec(..., seed, spread))."""
        el = np.ascontiguousarray(base.load_elements, dtype=np.int32)
        arrs = [np.ascontiguousarray(a, dtype=np.float64)
                for a in (base.p_load, base.q_load, base.p_gen, base.q_gen)]
        p = _out_array((count, self.n_theta), np.float64, device)
        q = _out_array((count, self.n_q), np.float64, device)
        flags = ACPF_DEVICE_PTRS if device is not None else ACPF_HOST_PTRS
        _check(_lib.acpf_nr_scenarios(self._h, int(seed), int(start), int(count), float(spread),
                                      el.size, _ptr(el), *[_ptr(a) for a in arrs], _ptr(p), _ptr(q),
                                      flags, None))
        return p, q

    def set_fd(self, y_csr, theta_block, q_block, epsilon: float = 1e-6) -> None:
        """Attach the fast-decoupled preconditioner data (acpf_nr_plan_set_fd):
        explicit inverses of B' + eps I and B'' + eps I (factorised with the
        reference's singularity test, sparse.py:159-183) and G = -Re Y[q, th]."""
        import scipy.linalg
        import scipy.sparse
        y = y_csr.tocsr()
        tb = np.asarray(theta_block, dtype=np.int64)
        qb = np.asarray(q_block, dtype=np.int64)

        def inverse(block):
            dense = -(y[block][:, block].imag).toarray()
            n = dense.shape[0]
            if n == 0:
                return np.zeros((0, 0))
            dense = dense + epsilon * np.eye(n)
            lu, piv = scipy.linalg.lu_factor(dense, check_finite=False)
            scale = max(np.abs(dense).max(), np.finfo(np.float64).tiny)
            if not np.all(np.isfinite(lu)) or np.abs(np.diag(lu)).min() <= n * np.finfo(np.float64).eps * scale:
                raise EngineError(f"block of dim {n} numerically singular (epsilon={epsilon!r})")
            return np.ascontiguousarray(scipy.linalg.lu_solve((lu, piv), np.eye(n), check_finite=False))

        b1, b2 = inverse(tb), inverse(qb)
        g = scipy.sparse.csr_matrix(-(y[qb][:, tb].real))
        g.eliminate_zeros()
        g.sort_indices()
        rp = np.ascontiguousarray(g.indptr, dtype=np.int32)
        col = np.ascontiguousarray(g.indices, dtype=np.int32)
        val = np.ascontiguousarray(g.data, dtype=np.float64)
        _check(_lib.acpf_nr_plan_set_fd(self._h, _ptr(b1) if b1.size else None, _ptr(b2) if b2.size else None,
                                        _ptr(rp), _ptr(col) if col.size else None,
                                        _ptr(val) if val.size else None))
        self._fd_eps = epsilon

    def solve_gmres(self, p_spec, q_spec, tol: float, max_newton: int, precond: str = "fd",
                    gmres_tol: float = 1e-8, restart: int = 60, max_outer: int = 10, stream=None,
                    out: dict | None = None) -> dict:
        """The reference's Newton step (matrix-free GMRES, FD or no
        preconditioner) for a stacked batch (acpf_nr_solve_gmres)."""
        dev = _is_device(p_spec)
        b = int(p_spec.shape[0])
        if out is not None:
            pass
        elif dev:
            out = self.alloc_outputs(b, like=p_spec)
            import torch
            kw = dict(device=p_spec.device)
            out["gmres_steps"] = torch.zeros((b, max_newton), dtype=torch.int32, **kw)
            out["gmres_diag"] = torch.zeros(b, dtype=torch.int32, **kw)
            out["gmres_diag_k"] = torch.zeros(b, dtype=torch.int32, **kw)
            out["gmres_diag_relres"] = torch.zeros(b, dtype=torch.float64, **kw)
        else:
            out = self.alloc_outputs(b)
            out["gmres_steps"] = np.zeros((b, max_newton), dtype=np.int32)
            out["gmres_diag"] = np.zeros(b, dtype=np.int32)
            out["gmres_diag_k"] = np.zeros(b, dtype=np.int32)
            out["gmres_diag_relres"] = np.zeros(b)
        flags = ACPF_DEVICE_PTRS if dev else ACPF_HOST_PTRS
        _check(_lib.acpf_nr_solve_gmres(
            self._h, b, _ptr(p_spec), _ptr(q_spec), float(tol), int(max_newton), float(gmres_tol),
            int(restart), int(max_outer), 1 if precond == "fd" else 0, _ptr(out["theta"]),
            _ptr(out["vmag"]), _ptr(out["converged"]), _ptr(out["iterations"]),
            _ptr(out["final_mismatch_inf"]), _ptr(out["status"]), _ptr(out["gmres_steps"]),
            _ptr(out["gmres_diag"]), _ptr(out["gmres_diag_k"]), _ptr(out["gmres_diag_relres"]), flags,
            _stream_ptr(stream)))
        return out

    def set_branches(self, net) -> None:
        """Attach the branch table (acpf_nr_plan_set_branches) for certify()."""
        f, t, y4, gs = branch_admittances(net)
        _check(_lib.acpf_nr_plan_set_branches(self._h, f.size, _ptr(f), _ptr(t), _ptr(y4), _ptr(gs)))
        self._branches = True

    def certify(self, theta, vmag, p_spec, q_spec, stream=None) -> dict:
        """Per-scenario certificates of solved states on the GPU
        (acpf_nr_certify): mismatch_inf, slack_balance, branch_loss."""
        dev = _is_device(theta)
        b = int(theta.shape[0])
        out = {k: _out_array((b,), np.float64, theta.device if dev else None)
               for k in ("mismatch_inf", "slack_balance", "branch_loss")}
        _check(_lib.acpf_nr_certify(
            self._h, b, _ptr(theta), _ptr(vmag), _ptr(p_spec) if self.n_theta else None,
            _ptr(q_spec) if self.n_q else None, _ptr(out["mismatch_inf"]), _ptr(out["slack_balance"]),
            _ptr(out["branch_loss"]), ACPF_DEVICE_PTRS if dev else ACPF_HOST_PTRS, _stream_ptr(stream)))
        return out

    def close(self) -> None:
        if getattr(self, "_h", None) and _lib is not None:
            _lib.acpf_nr_plan_destroy(self._h)
            self._h = None

    __del__ = close


# ---------------------------------------------------------------------------
# Z-Bus plans
# ---------------------------------------------------------------------------


class ZbusPlan:
    """Device plan for one feeder (acpf_zbus_plan_create)."""

    def __init__(self, model, device: int = 0):
        require_device(device)
        lib = load_library()
        self.n = int(model.n)
        self.n_wye = int(model.wye_idx.size)
        self.n_delta = int(model.delta_p.size)
        cols = np.ascontiguousarray(model.load_cols, dtype=np.int32)
        zl = np.ascontiguousarray(model.z_load, dtype=np.complex128)
        v0 = np.ascontiguousarray(model.v0, dtype=np.complex128)
        wi = np.ascontiguousarray(model.wye_idx, dtype=np.int32)
        dp = np.ascontiguousarray(model.delta_p, dtype=np.int32)
        dq = np.ascontiguousarray(model.delta_q, dtype=np.int32)
        h = P()
        _check(lib.acpf_zbus_plan_create(device, self.n, cols.size, _ptr(cols), _ptr(zl), _ptr(v0),
                                         wi.size, _ptr(wi), dp.size, _ptr(dp), _ptr(dq),
                                         float(model.voltage_floor), C.byref(h)))
        self._h = h
        self.device = device

    def alloc_outputs(self, b: int, like=None) -> dict:
        if like is not None:
            import torch
            kw = dict(device=like.device)
            return {
                "v": torch.empty((b, self.n), dtype=torch.complex128, **kw),
                "converged": torch.empty(b, dtype=torch.uint8, **kw),
                "iterations": torch.empty(b, dtype=torch.int32, **kw),
                "final_delta": torch.empty(b, dtype=torch.float64, **kw),
                "residual_inf": torch.empty(b, dtype=torch.float64, **kw),
                "status": torch.empty(b, dtype=torch.int32, **kw),
                "floor_slot": torch.empty(b, dtype=torch.int32, **kw),
            }
        from . import hostmem
        return {
            "v": hostmem.empty((b, self.n), np.complex128),
            "converged": hostmem.empty(b, np.uint8), "iterations": hostmem.empty(b, np.int32),
            "final_delta": hostmem.empty(b), "residual_inf": hostmem.empty(b),
            "status": hostmem.empty(b, np.int32), "floor_slot": hostmem.empty(b, np.int32),
        }

    def solve(self, s_wye, s_delta, tol: float, max_iter: int, out: dict | None = None,
              stream=None) -> dict:
        dev = _is_device(s_wye)
        b = int(s_wye.shape[0])
        if out is None:
            out = self.alloc_outputs(b, like=s_wye if dev else None)
        flags = ACPF_DEVICE_PTRS if dev else ACPF_HOST_PTRS
        _check(_lib.acpf_zbus_solve(
            self._h, b, _ptr(s_wye) if self.n_wye else None,
            _ptr(s_delta) if self.n_delta else None, float(tol), int(max_iter), _ptr(out["v"]),
            _ptr(out["converged"]), _ptr(out["iterations"]), _ptr(out["final_delta"]),
            _ptr(out["residual_inf"]), _ptr(out["status"]), _ptr(out["floor_slot"]), flags,
            _stream_ptr(stream, s_wye)))
        return out

    def last_timing(self) -> tuple:
        ms, n = D(), I32()
        _check(_lib.acpf_zbus_last_timing(self._h, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def scenarios(self, base, seed: int, start: int, count: int, spread: float = 0.2, device=None):
        """Seeded (s_wye, s_delta) rows generated on the GPU, bitwise
        batch.make_scenario_arrays(base, ScenarioSpec(..., target='distribution'))."""
        kinds = list(base.load_kinds)
        tgt, wi, di = [], 0, 0
        for k in kinds:
            if k == "wye":
                tgt.append(wi)
                wi += 1
            else:
                tgt.append(-di - 1)
                di += 1
        tgt = np.ascontiguousarray(tgt, dtype=np.int32)
        ws = np.ascontiguousarray(base.wye_s, dtype=np.complex128)
        ds = np.ascontiguousarray(base.delta_s, dtype=np.complex128)
        sw = _out_array((count, self.n_wye), np.complex128, device)
        sd = _out_array((count, self.n_delta), np.complex128, device)
        flags = ACPF_DEVICE_PTRS if device is not None else ACPF_HOST_PTRS
        _check(_lib.acpf_zbus_scenarios(self._h, int(seed), int(start), int(count), float(spread),
                                        tgt.size, _ptr(tgt), _ptr(ws) if ws.size else None,
                                        _ptr(ds) if ds.size else None,
                                        _ptr(sw) if self.n_wye else None,
                                        _ptr(sd) if self.n_delta else None, flags, None))
        return sw, sd

    def set_network(self, model) -> None:
        """Attach Y_NN and Y_NS v_slack (acpf_zbus_plan_set_network) for kirchhoff()."""
        y = model.y_nn.tocsr()
        y.sort_indices()
        rp = np.ascontiguousarray(y.indptr, dtype=np.int32)
        col = np.ascontiguousarray(y.indices, dtype=np.int32)
        val = np.ascontiguousarray(y.data, dtype=np.complex128)
        inj = np.ascontiguousarray(model.y_ns @ model.v_slack, dtype=np.complex128)
        _check(_lib.acpf_zbus_plan_set_network(self._h, _ptr(rp), _ptr(col) if col.size else None,
                                               _ptr(val) if val.size else None, _ptr(inj)))
        self._network = True

    def kirchhoff(self, v, s_wye, s_delta, stream=None):
        """max_k |Y_NN v + Y_NS v_s - i_loads(v)| per scenario (acpf_zbus_kirchhoff);
        inf where a load voltage is at the floor."""
        dev = _is_device(v)
        b = int(v.shape[0])
        out = _out_array((b,), np.float64, v.device if dev else None)
        _check(_lib.acpf_zbus_kirchhoff(
            self._h, b, _ptr(v), _ptr(s_wye) if self.n_wye else None,
            _ptr(s_delta) if self.n_delta else None, _ptr(out),
            ACPF_DEVICE_PTRS if dev else ACPF_HOST_PTRS, _stream_ptr(stream)))
        return out

    def close(self) -> None:
        if getattr(self, "_h", None) and _lib is not None:
            _lib.acpf_zbus_plan_destroy(self._h)
            self._h = None

    __del__ = close


def zbus_reduce(y_nn, rhs0, l_index, device: int = 0):
    """Y_NN^-1 [E_l | rhs0] on the GPU (acpf_zbus_reduce): (Z[:, l], v0).
    Raises EngineError with the reference's singular-Ybus text when Y_NN is
    numerically singular (status ACPF_ESTRUCT)."""
    require_device(device)
    lib = load_library()
    y = y_nn.tocsr()
    y.sort_indices()
    n = y.shape[0]
    rp = np.ascontiguousarray(y.indptr, dtype=np.int32)
    col = np.ascontiguousarray(y.indices, dtype=np.int32)
    val = np.ascontiguousarray(y.data, dtype=np.complex128)
    r0 = np.ascontiguousarray(rhs0, dtype=np.complex128)
    li = np.ascontiguousarray(l_index, dtype=np.int32)
    zl = np.empty((n, li.size), dtype=np.complex128)
    v0 = np.empty(n, dtype=np.complex128)
    _check(lib.acpf_zbus_reduce(device, n, _ptr(rp), _ptr(col) if col.size else None,
                                _ptr(val) if val.size else None, _ptr(r0), li.size,
                                _ptr(li) if li.size else None, _ptr(zl) if li.size else None, _ptr(v0)))
    return zl, v0


def zbus_plan_for(model, device: int | None = None, slot: int = 0) -> ZbusPlan:
    """The model's plan on ``device`` (one per (device, slot): a plan is driven
    by one host thread at a time, include/acpf.h)."""
    device = 0 if device is None else device
    key = device if slot == 0 else (device, slot)
    plan = model._plans.get(key)
    if plan is None:
        plan = ZbusPlan(model, device)
        model._plans[key] = plan
    return plan


def zbus_solve_arrays(model, s_wye, s_delta, tol, max_iter, device=None) -> dict:
    plan = zbus_plan_for(model, device)
    sw = np.ascontiguousarray(s_wye, dtype=np.complex128)
    sd = np.ascontiguousarray(s_delta, dtype=np.complex128)
    if sd.size == 0:
        sd = np.zeros((sw.shape[0], 0), dtype=np.complex128)
    return plan.solve(sw, sd, tol, max_iter)


def zbus_floor_message(model, v: np.ndarray, slot: int) -> str:
    """Reconstruct the reference VoltageFloorError text (distribution.py:45-50)."""
    from .distribution import floor_site_label
    nw, nd = model.wye_idx.size, model.delta_p.size
    if slot < nw:
        kind, k, mag = "wye", slot, abs(v[model.wye_idx[slot]])
    elif slot < nw + nd:
        k = slot - nw
        kind, mag = "p", abs(v[model.delta_p[k]])
    elif slot < nw + 2 * nd:
        k = slot - nw - nd
        kind, mag = "q", abs(v[model.delta_q[k]])
    else:
        k = slot - nw - 2 * nd
        kind, mag = "pq", abs(v[model.delta_p[k]] - v[model.delta_q[k]])
    label = floor_site_label(model, kind, k)
    return f"voltage magnitude {float(mag):.3e} below floor at node-phase {label}"


def zbus_results(model, out: dict) -> list:
    """FixedPointResult records of stacked Z-Bus outputs (results.ZbusResults)."""
    from .results import ZbusResults
    return list(ZbusResults(model, out))


@dataclass
class Timing:
    kernel_ms: float
    launches: int
