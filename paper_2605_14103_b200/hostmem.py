"""Page-locked host arrays for the host-pointer solves.

The C-ABI copies a host batch in and the results out on its own streams
(acpf_nr_solve / acpf_zbus_solve with ACPF_HOST_PTRS). From pageable memory
those copies are staged by the driver and block the issuing thread, which
serialises them with the solve; from page-locked memory they run at PCIe
rate and overlap the other chunk's solve. Scenario tables built by
``make_scenario_arrays`` and result tables allocated by the solvers therefore
come from torch's caching pinned-host allocator (buffers are recycled when
the arrays are released). Without a CUDA device this is plain numpy.
"""

from __future__ import annotations

import numpy as np

_state = {"ok": None}


def _pinned_available() -> bool:
    if _state["ok"] is None:
        try:
            import torch
            _state["ok"] = bool(torch.cuda.is_available())
        except Exception:
            _state["ok"] = False
    return _state["ok"]


def empty(shape, dtype=np.float64) -> np.ndarray:
    """Uninitialised host array, page-locked when a CUDA device is present."""
    dtype = np.dtype(dtype)
    if not _pinned_available():
        return np.empty(shape, dtype=dtype)
    import torch
    n = int(np.prod(shape, dtype=np.int64)) * dtype.itemsize
    buf = torch.empty(max(n, 1), dtype=torch.uint8, pin_memory=True).numpy()
    return buf[:n].view(dtype).reshape(shape)
