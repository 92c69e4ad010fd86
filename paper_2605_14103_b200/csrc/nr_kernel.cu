// Batched polar Newton-Raphson on sm_100a: one warp = 32 scenarios in
// lock-step, lane = scenario, every per-scenario array interleaved
// [row][32] so each warp access is one coalesced 256-byte transaction and
// the shared schedule (Ybus, LU pattern, Crout pairs) is a warp-uniform
// broadcast load.
//
// One launch runs the whole Newton loop of the reference `_newton_loop`
// (transmission.py:333-380) for its warp's scenarios, with no host round
// trip:
//   A  phasors      u = V e^{j theta}                  (transmission.py:196)
//   B  mismatch     I = Y u, S = u conj(I), F, ||F||inf (transmission.py:194-215)
//      exit checks in the reference order: non-finite -> converged ->
//      min V <= 0 -> k == max_newton                  (transmission.py:347-359)
//   C  Jacobian assembly fused into a Crout (row-by-row, dot-product form)
//      static-pivot LU refactorisation, forward substitution fused
//      (replaces the GMRES/FD step of transmission.py:361-369)
//   D  back substitution and x += dx                   (transmission.py:378)
// Jacobian entries are produced on the fly from the Ybus entry that feeds
// each LU slot (the block formulas of dense_jacobian, transmission.py:383-407),
// so the factor storage is written exactly once per slot per Newton step.

#include "acpf_internal.cuh"

namespace acpf {

namespace {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// u_i * conj(a)
__device__ __forceinline__ double2 mul_conj(double2 u, double2 a) {
  return make_double2(u.x * a.x + u.y * a.y, u.y * a.x - u.x * a.y);
}

__global__ void __launch_bounds__(128) nr_newton_kernel(NrDeviceModel m, NrWorkspace w,
                                                        NrBatchIO io, double tol,
                                                        int max_newton) {
  const int lane = threadIdx.x & 31;
  const int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (g >= w.groups) return;
  const int64_t s = g * kGroup + lane;
  const bool valid = s < io.batch;

  const int64_t ws_lu = g * m.nnz_lu * kGroup;
  double* __restrict__ lu = w.lu + ws_lu + lane;
  double* __restrict__ invd = w.invd + g * m.n_j * kGroup + lane;
  double* __restrict__ yx = w.yx + g * m.n_j * kGroup + lane;
  double* __restrict__ spec = w.spec + g * m.n_j * kGroup + lane;
  double* __restrict__ th = w.th + g * m.n_bus * kGroup + lane;
  double* __restrict__ vm = w.vm + g * m.n_bus * kGroup + lane;
  double2* __restrict__ U = w.U + g * m.n_bus * kGroup + lane;
  double2* __restrict__ E = w.E + g * m.n_bus * kGroup + lane;
  double2* __restrict__ I = w.I + g * m.n_bus * kGroup + lane;

  // flat start + interleave this lane's specified injections
  for (int i = 0; i < m.n_bus; ++i) {
    th[i * kGroup] = m.theta_init[i];
    vm[i * kGroup] = m.vmag_init[i];
  }
  for (int r = 0; r < m.n_j; ++r) {
    double v = 0.0;
    if (valid)
      v = r < m.n_theta ? io.p_spec[s * m.n_theta + r] : io.q_spec[s * m.n_q + (r - m.n_theta)];
    spec[r * kGroup] = v;
  }

  bool done = !valid;
  int status = 0, iters = 0;
  double fout = 0.0;

  for (int k = 0; k <= max_newton; ++k) {
    // ---- A: phasors, min V
    double vmin = __longlong_as_double(0x7ff0000000000000LL);  // +inf
    for (int i = 0; i < m.n_bus; ++i) {
      const double t = th[i * kGroup], v = vm[i * kGroup];
      double sn, cs;
      sincos(t, &sn, &cs);
      E[i * kGroup] = make_double2(cs, sn);
      U[i * kGroup] = make_double2(v * cs, v * sn);
      vmin = fmin(vmin, v);
    }
    // ---- B: injections and mismatch
    double fmax = 0.0;
    bool anynan = false, anyinf = false;
    for (int i = 0; i < m.n_bus; ++i) {
      double2 acc = make_double2(0.0, 0.0);
      const int e1 = m.y_rowptr[i + 1];
      for (int e = m.y_rowptr[i]; e < e1; ++e) {
        const double2 y = m.y_val[e];
        const double2 u = U[m.y_col[e] * kGroup];
        acc.x += y.x * u.x - y.y * u.y;
        acc.y += y.x * u.y + y.y * u.x;
      }
      I[i * kGroup] = acc;
      const double2 ui = U[i * kGroup];
      const double2 sc = mul_conj(ui, acc);  // S_i = u_i conj(I_i)
      const int tp = m.tpos[i], qp = m.qpos[i];
      if (tp >= 0) {
        const double f = sc.x - spec[tp * kGroup];
        anynan |= isnan(f);
        anyinf |= isinf(f);
        fmax = fmax < fabs(f) ? fabs(f) : fmax;
        yx[m.ipos[tp] * kGroup] = -f;
      }
      if (qp >= 0) {
        const double f = sc.y - spec[qp * kGroup];
        anynan |= isnan(f);
        anyinf |= isinf(f);
        fmax = fmax < fabs(f) ? fabs(f) : fmax;
        yx[m.ipos[qp] * kGroup] = -f;
      }
    }
    if (!done) {
      if (anynan || anyinf) {
        done = true;
        status = ACPF_NR_NONFINITE;
        iters = k;
        fout = anynan ? __longlong_as_double(0x7ff8000000000000LL) : fmax;
      } else if (fmax <= tol) {
        done = true;
        status = ACPF_NR_CONVERGED;
        iters = k;
        fout = fmax;
      } else if (vmin <= 0.0) {
        done = true;
        status = ACPF_NR_VMAG_LE0;
        iters = k;
        fout = fmax;
      } else if (k == max_newton) {
        done = true;
        status = ACPF_NR_MAX_ITER;
        iters = max_newton;
        fout = fmax;
      }
    }
    if (__all_sync(0xffffffffu, done)) break;

    // ---- C: assembly + Crout refactorisation + forward substitution
    bool zero_pivot = false;
    for (int p = 0; p < m.n_j; ++p) {
      const int bi = m.row_bus[p];
      const double2 ui = U[bi * kGroup];
      const double2 Ii = I[bi * kGroup];
      const int t0 = m.lu_rowptr[p], t1 = m.lu_rowptr[p + 1], td = m.lu_diag[p];
      double yacc = yx[p * kGroup];
      for (int t = t0; t < t1; ++t) {
        const int2 d = m.slot_desc[t];
        const int type = (unsigned)d.y >> 28;
        double a = 0.0;
        if (type < 8) {
          const int j = d.y & 0x0fffffff;
          const double2 y = d.x >= 0 ? m.y_val[d.x] : make_double2(0.0, 0.0);
          const bool diag = type & 4, qrow = type & 2;
          if (type & 1) {  // d/dV_j: u_i conj(y E_j) [+ conj(I_i) E_i]
            const double2 ej = E[j * kGroup];
            const double2 wv = mul_conj(ui, cmul(y, ej));
            if (!diag) {
              a = qrow ? wv.y : wv.x;
            } else {
              a = qrow ? wv.y + (Ii.x * ej.y - Ii.y * ej.x) : wv.x + (Ii.x * ej.x + Ii.y * ej.y);
            }
          } else {  // d/dtheta_j
            if (!diag) {  // -j u_i conj(y u_j)
              const double2 wv = mul_conj(ui, cmul(y, U[j * kGroup]));
              a = qrow ? -wv.x : wv.y;
            } else {  // j u_i conj(I_i - y u_i)
              const double2 yu = cmul(y, ui);
              const double2 wv = mul_conj(ui, make_double2(Ii.x - yu.x, Ii.y - yu.y));
              a = qrow ? wv.x : -wv.y;
            }
          }
        }
        const int q1 = m.pair_ptr[t + 1];
#pragma unroll 4
        for (int q = m.pair_ptr[t]; q < q1; ++q) {
          const int2 pr = m.pairs[q];
          a = fma(-lu[pr.x * kGroup], lu[pr.y * kGroup], a);
        }
        if (t < td) {
          const int c = m.lu_col[t];
          a *= invd[c * kGroup];
          yacc = fma(-a, yx[c * kGroup], yacc);
        } else if (t == td) {
          zero_pivot |= (a == 0.0);
          invd[p * kGroup] = 1.0 / a;
        }
        lu[t * kGroup] = a;
      }
      yx[p * kGroup] = yacc;
    }
    // ---- D: back substitution
    for (int p = m.n_j - 1; p >= 0; --p) {
      double acc = yx[p * kGroup];
      const int t1 = m.lu_rowptr[p + 1];
      for (int t = m.lu_diag[p] + 1; t < t1; ++t) acc = fma(-lu[t * kGroup], yx[m.lu_col[t] * kGroup], acc);
      yx[p * kGroup] = acc * invd[p * kGroup];
    }
    if (!done && zero_pivot) {
      done = true;
      status = ACPF_NR_ZERO_PIVOT;
      iters = k;
      fout = fmax;
    }
    if (!done) {
      for (int i = 0; i < m.n_bus; ++i) {
        const int tp = m.tpos[i], qp = m.qpos[i];
        if (tp >= 0) th[i * kGroup] = th[i * kGroup] + yx[m.ipos[tp] * kGroup];
        if (qp >= 0) vm[i * kGroup] = vm[i * kGroup] + yx[m.ipos[qp] * kGroup];
      }
    }
  }

  if (!valid) return;
  for (int i = 0; i < m.n_bus; ++i) {
    io.theta_out[s * m.n_bus + i] = th[i * kGroup];
    io.vmag_out[s * m.n_bus + i] = vm[i * kGroup];
  }
  if (io.converged) io.converged[s] = status == ACPF_NR_CONVERGED;
  if (io.iterations) io.iterations[s] = iters;
  if (io.fnorm) io.fnorm[s] = fout;
  if (io.status) io.status[s] = status;
}

}  // namespace

cudaError_t launch_nr_newton(const NrDeviceModel& m, const NrWorkspace& w, const NrBatchIO& io,
                             double tol, int max_newton, cudaStream_t stream) {
  const int warps_per_block = 4;
  const int64_t blocks = (w.groups + warps_per_block - 1) / warps_per_block;
  nr_newton_kernel<<<(unsigned)blocks, 32 * warps_per_block, 0, stream>>>(m, w, io, tol, max_newton);
  return cudaGetLastError();
}

}  // namespace acpf
