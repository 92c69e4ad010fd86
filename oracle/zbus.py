"""Z-Bus oracle: restatement of the reference fixed point (distribution.py).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.linalg


@dataclass
class ZbCase:
    y_nn: object            # non-slack block (distribution.py:457)
    v0: np.ndarray          # no-load profile (:474)
    wye_idx: np.ndarray     # reduced indices (:480-499)
    delta_p: np.ndarray
    delta_q: np.ndarray
    voltage_floor: float = 1e-6

    def __post_init__(self):
        self.n = int(self.v0.size)
        dense = self.y_nn.toarray()
        self.lu = scipy.linalg.lu_factor(dense, check_finite=False)  # (:463)

    def z_apply(self, w):
        """Y_NN^{-1} w by LU solve (distribution.py:423-425)."""
        return scipy.linalg.lu_solve(self.lu, w, check_finite=False)


class Floor(Exception):
    def __init__(self, slot):
        self.slot = slot


def injection(case: ZbCase, v, s_wye, s_delta):
    """Load currents (distribution.py:573-610): wye -conj(s/v_p), then delta
    line currents conj(s/(v_p-v_q)) subtracted at p and added at q, np.add.at
    order; floor checks wye, delta p, delta q, p-q. Raises Floor(slot) with the
    C-ABI floor_slot numbering."""
    i = np.zeros(case.n, dtype=np.complex128)
    fl = case.voltage_floor
    nw, nd = case.wye_idx.size, case.delta_p.size
    if nw:
        bad = np.flatnonzero(np.abs(v[case.wye_idx]) <= fl)
        if bad.size:
            raise Floor(int(bad[0]))
        np.add.at(i, case.wye_idx, -np.conj(s_wye / v[case.wye_idx]))
    if nd:
        vp, vq = v[case.delta_p], v[case.delta_q]
        for base, arr in ((nw, vp), (nw + nd, vq), (nw + 2 * nd, vp - vq)):
            bad = np.flatnonzero(np.abs(arr) <= fl)
            if bad.size:
                raise Floor(base + int(bad[0]))
        il = np.conj(s_delta / (vp - vq))
        np.add.at(i, case.delta_p, -il)
        np.add.at(i, case.delta_q, il)
    return i


@dataclass
class ZbOut:
    v: np.ndarray
    converged: bool
    iterations: int
    final_delta: float
    residual_inf: float
    floor_slot: int


def zbus(case: ZbCase, s_wye, s_delta, tol=1e-9, max_iter=100) -> ZbOut:
    """_zbus_loop (distribution.py:653-687) + fixed_point_residual (:613-621)."""
    v = case.v0.copy()
    mag = float(np.abs(v).sum())
    delta = float("inf")
    converged = False
    k = 0
    for k in range(1, max_iter + 1):
        try:
            i = injection(case, v, s_wye, s_delta)
        except Floor as fl:
            return ZbOut(v, False, k, delta, float("inf"), fl.slot)
        v = case.z_apply(i) + case.v0
        s = float(np.abs(v).sum())
        delta = abs(s - mag)
        mag = s
        if delta <= tol:
            converged = True
            break
    try:
        res = float(np.abs(v - (case.z_apply(injection(case, v, s_wye, s_delta)) + case.v0)).max())
    except Floor:
        res = float("inf")
    return ZbOut(v, converged, k, delta, res, -1)
