"""Newton-Raphson oracle: restatement of the reference's GMRES-FD Newton.

Reference: pkg/src/acpflow/transmission.py and sparse.py. The model inputs
(Y-bus, partition, flat start) come from the host loader, whose Y-bus is
pinned bitwise to the reference by tests/test_host_model.py.
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.linalg
import scipy.sparse
import scipy.sparse.linalg

NONFINITE = "mismatch became non-finite (diverged iterate)"  # transmission.py:351
COLLAPSE = "voltage magnitude iterate collapsed to <= 0 (diverging)"  # transmission.py:356


@dataclass
class NrCase:
    """What the oracle needs from a transmission model."""

    y: scipy.sparse.csr_matrix  # complex Ybus (network.py:450-496)
    theta_block: np.ndarray     # PV then PQ (network.py:499-516)
    q_block: np.ndarray         # PQ
    theta0: np.ndarray          # flat start (transmission.py:169-177)
    vmag0: np.ndarray
    epsilon: float = 1e-6       # NewtonOptions.epsilon (transmission.py:104)

    def __post_init__(self):
        self.y = self.y.tocsr()
        self._fd = None

    @property
    def n_theta(self) -> int:
        return int(self.theta_block.size)

    # --- FD factors: B' = -Im Y[th,th], B'' = -Im Y[q,q], G = -Re Y[q,th]
    #     (network.py:519-543), factorised once with eps*I (transmission.py:259-266,
    #     sparse.py:159-183)
    def fd(self):
        if self._fd is None:
            tb, qb = self.theta_block, self.q_block
            bp = -(self.y[tb][:, tb].imag).toarray()
            bpp = -(self.y[qb][:, qb].imag).toarray()
            g = scipy.sparse.csr_matrix(-(self.y[qb][:, tb].real))
            g.eliminate_zeros()
            f1 = scipy.linalg.lu_factor(bp + self.epsilon * np.eye(bp.shape[0]), check_finite=False)
            f2 = (scipy.linalg.lu_factor(bpp + self.epsilon * np.eye(bpp.shape[0]), check_finite=False)
                  if bpp.size else None)
            self._fd = (f1, f2, g)
        return self._fd


def injections(y, theta, vmag):
    """P, Q at every bus: u = V e^{j theta}, S = u conj(Y u) (transmission.py:194-199)."""
    u = vmag * np.exp(1j * theta)
    s = u * np.conj(y @ u)
    return s.real, s.imag


def mismatch(case: NrCase, theta, vmag, p_spec, q_spec):
    """F over the theta block then the PQ block (transmission.py:202-215)."""
    p, q = injections(case.y, theta, vmag)
    return np.concatenate([p[case.theta_block] - p_spec, q[case.q_block] - q_spec])


def _jvp(case: NrCase, theta, vmag):
    """dF = J dx via du = e^{j th} dV + j u dth, dS = du conj(I) + u conj(Y du)
    (transmission.py:218-236)."""
    ph = np.exp(1j * theta)
    u = vmag * ph
    ic = np.conj(case.y @ u)
    nt, n = case.n_theta, theta.size
    tb, qb = case.theta_block, case.q_block

    def op(dx):
        dth = np.zeros(n)
        dvm = np.zeros(n)
        dth[tb] = dx[:nt]
        dvm[qb] = dx[nt:]
        du = ph * dvm + 1j * u * dth
        ds = du * ic + u * np.conj(case.y @ du)
        return np.concatenate([ds.real[tb], ds.imag[qb]])

    return op


def _precond(case: NrCase, vmag):
    """Forward block substitution with the fixed FD factors and voltage
    scalings (transmission.py:269-298)."""
    f1, f2, g = case.fd()
    vt, vq = vmag[case.theta_block], vmag[case.q_block]
    nt = case.n_theta

    def apply(rv):
        zt = scipy.linalg.lu_solve(f1, rv[:nt] / vt, check_finite=False)
        rq = (rv[nt:] - g @ zt) / vq
        zq = scipy.linalg.lu_solve(f2, rq, check_finite=False) if f2 is not None else rq
        return np.concatenate([zt, zq])

    return apply


def gmres(op, pre, rhs, tol=1e-8, restart=60, max_outer=10):
    """Left-preconditioned restarted GMRES, MGS + Givens, zero start
    (sparse.py:219-338). Returns (x, iterations, converged, breakdown, relres)."""
    n = rhs.size
    mb = pre(rhs)
    if not np.all(np.isfinite(mb)):
        raise FloatingPointError("preconditioner produced non-finite values")
    beta0 = float(np.linalg.norm(mb))
    if beta0 == 0.0:
        return np.zeros(n), 0, True, False, 0.0
    x = np.zeros(n)
    total = 0
    breakdown = converged = False
    relres = 1.0
    m = min(restart, n)
    for cycle in range(max_outer + 1):
        r = mb.copy() if cycle == 0 else pre(rhs - op(x))
        beta = float(np.linalg.norm(r))
        relres = beta / beta0
        if relres <= tol:
            converged = True
            break
        if cycle == max_outer or breakdown:
            break
        basis = np.empty((m + 1, n))
        h = np.zeros((m + 1, m))
        cs = np.zeros(m)
        sn = np.zeros(m)
        gv = np.zeros(m + 1)
        gv[0] = beta
        basis[0] = r / beta
        k = 0
        for j in range(m):
            w = np.array(pre(op(basis[j])), dtype=np.float64)
            for i in range(j + 1):
                h[i, j] = basis[i] @ w
                w -= h[i, j] * basis[i]
            hn = float(np.linalg.norm(w))
            h[j + 1, j] = hn
            for i in range(j):
                t = cs[i] * h[i, j] + sn[i] * h[i + 1, j]
                h[i + 1, j] = -sn[i] * h[i, j] + cs[i] * h[i + 1, j]
                h[i, j] = t
            den = float(np.hypot(h[j, j], h[j + 1, j]))
            if den == 0.0:
                breakdown = True
                k = j
                break
            cs[j] = h[j, j] / den
            sn[j] = h[j + 1, j] / den
            h[j, j] = den
            h[j + 1, j] = 0.0
            gv[j + 1] = -sn[j] * gv[j]
            gv[j] = cs[j] * gv[j]
            total += 1
            k = j + 1
            rel = abs(gv[j + 1]) / beta0
            if hn <= 1e-14 * beta0:
                if rel > tol:
                    breakdown = True
                break
            if rel <= tol:
                break
            basis[j + 1] = w / hn
        yv = np.zeros(k)
        for i in range(k - 1, -1, -1):
            yv[i] = (gv[i] - h[i, i + 1:k] @ yv[i + 1:k]) / h[i, i]
        x = x + basis[:k].T @ yv
    return x, total, converged, breakdown, relres


@dataclass
class NrOut:
    theta: np.ndarray
    vmag: np.ndarray
    converged: bool
    iterations: int
    final_mismatch_inf: float
    diagnostic: str | None


def newton(case: NrCase, p_spec, q_spec, tol=1e-8, max_newton=20, step="gmres") -> NrOut:
    """The reference Newton driver _newton_loop (transmission.py:333-380).

    Exit checks per iterate, in order: non-finite mismatch, ||F||inf <= tol,
    min V <= 0, k == max_newton; else step and x += dx. ``step='gmres'`` is the
    reference's FD-preconditioned GMRES; ``step='lu'`` an exact sparse-LU step
    (same driver) for fast cross-checks."""
    theta, vmag = case.theta0.copy(), case.vmag0.copy()
    tb, qb, nt = case.theta_block, case.q_block, case.n_theta
    diag = None
    fnorm = np.inf
    for k in range(max_newton + 1):
        f = mismatch(case, theta, vmag, p_spec, q_spec)
        fnorm = float(np.abs(f).max()) if f.size else 0.0
        if not np.isfinite(fnorm):
            return NrOut(theta, vmag, False, k, fnorm, NONFINITE)
        if fnorm <= tol:
            return NrOut(theta, vmag, True, k, fnorm, diag)
        if vmag.size and vmag.min() <= 0.0:
            return NrOut(theta, vmag, False, k, fnorm, COLLAPSE)
        if k == max_newton:
            break
        if step == "gmres":
            dx, its, conv, brk, rr = gmres(_jvp(case, theta, vmag), _precond(case, vmag), -f)
            if brk:
                diag = f"GMRES breakdown at Newton iteration {k}"
            elif not conv and diag is None:
                diag = f"GMRES stagnated at Newton iteration {k} (relres {rr:.2e})"
        else:
            dx = scipy.sparse.linalg.spsolve(sparse_jacobian(case, theta, vmag).tocsc(), -f)
        x = np.concatenate([theta[tb], vmag[qb]]) + dx
        theta = theta.copy()
        vmag = vmag.copy()
        theta[tb] = x[:nt]
        vmag[qb] = x[nt:]
    return NrOut(theta, vmag, False, max_newton, fnorm, diag)


def sparse_jacobian(case: NrCase, theta, vmag):
    """J blocks H,N,M,L from the complex-form formulas of dense_jacobian
    (transmission.py:383-407), assembled sparse."""
    y = case.y
    e = np.exp(1j * theta)
    u = vmag * e
    i = y @ u
    du = scipy.sparse.diags(u)
    de = scipy.sparse.diags(e)
    dth = 1j * du @ np.conj(scipy.sparse.diags(i) - y @ du)
    dv = du @ np.conj(y @ de) + np.conj(scipy.sparse.diags(i)) @ de
    dth = scipy.sparse.csr_matrix(dth)
    dv = scipy.sparse.csr_matrix(dv)
    tb, qb = case.theta_block, case.q_block
    return scipy.sparse.bmat([[dth.real[tb][:, tb], dv.real[tb][:, qb]],
                              [dth.imag[qb][:, tb], dv.imag[qb][:, qb]]]).tocsr()
