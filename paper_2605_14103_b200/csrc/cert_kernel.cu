// On-device solution certificates.
//
// * NR: for each scenario's returned state (theta, V):
//     - ||F||inf recomputed from scratch (reference `mismatch`, transmission.py:202-215),
//     - the slack power balance of test_transmission.py:398-416:
//         sum_{slack} P_calc - (-sum_{theta block} p_spec + branch loss + shunt loss)
//       with the branch loss from per-branch flows (`branch_flows`,
//       transmission.py:453-481) — independent of the Ybus the solver used,
//     - the branch loss sum_br Re(s_from + s_to).
// * Z-Bus: the Kirchhoff residual max_k |(Y_NN v + Y_NS v_s)_k - i_loads(v)_k|
//   (`kirchhoff_residual`, distribution.py:624-630) with the sparse Y_NN.
//
// One CTA per scenario: the state is staged once in shared memory (u = V e^{j
// theta} or v), rows and branches are strided over the threads, and every
// reduction is a fixed-order tree, so results do not depend on the batch.

#include "acpf_internal.cuh"

namespace acpf {

namespace {

constexpr int kCertThreads = 256;

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// u * conj(a)
__device__ __forceinline__ double2 mul_conj(double2 u, double2 a) {
  return make_double2(u.x * a.x + u.y * a.y, u.y * a.x - u.x * a.y);
}

// a / b (Smith's scaling)
__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
  if (fabs(b.x) >= fabs(b.y)) {
    const double r = b.y / b.x, d = b.x + b.y * r;
    return make_double2((a.x + a.y * r) / d, (a.y - a.x * r) / d);
  }
  const double r = b.x / b.y, d = b.x * r + b.y;
  return make_double2((a.x * r + a.y) / d, (a.y * r - a.x) / d);
}

// fixed-order block reductions over kCertThreads values
__device__ double block_sum(double v, double* red) {
  const int t = threadIdx.x;
  red[t] = v;
  __syncthreads();
  for (int s = kCertThreads / 2; s > 0; s >>= 1) {
    if (t < s) red[t] = red[t] + red[t + s];
    __syncthreads();
  }
  const double r = red[0];
  __syncthreads();
  return r;
}

// max that propagates NaN (numpy max semantics)
__device__ __forceinline__ double nanmax(double a, double b) {
  return (isnan(a) || isnan(b)) ? __longlong_as_double(0x7ff8000000000000LL) : (a > b ? a : b);
}

__device__ double block_max(double v, double* red) {
  const int t = threadIdx.x;
  red[t] = v;
  __syncthreads();
  for (int s = kCertThreads / 2; s > 0; s >>= 1) {
    if (t < s) red[t] = nanmax(red[t], red[t + s]);
    __syncthreads();
  }
  const double r = red[0];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kCertThreads) nr_cert_kernel(NrCertModel m, NrCertIO io) {
  extern __shared__ __align__(16) unsigned char smem[];
  double2* u = reinterpret_cast<double2*>(smem);
  double* red = reinterpret_cast<double*>(u + m.n_bus);
  const int64_t s = blockIdx.x;
  const int t = threadIdx.x;
  const double* th = io.theta + s * m.n_bus;
  const double* vm = io.vmag + s * m.n_bus;
  double shunt = 0.0;
  for (int i = t; i < m.n_bus; i += kCertThreads) {
    double sn, cs;
    sincos(th[i], &sn, &cs);
    const double v = vm[i];
    u[i] = make_double2(v * cs, v * sn);
    shunt += m.gs[i] * v * v;
  }
  __syncthreads();
  double fmx = 0.0, pslack = 0.0, pspec = 0.0;
  for (int i = t; i < m.n_bus; i += kCertThreads) {
    double2 acc = make_double2(0.0, 0.0);
    for (int e = m.y_rowptr[i]; e < m.y_rowptr[i + 1]; ++e) {
      const double2 y = m.y_val[e], uj = u[m.y_col[e]];
      acc.x += y.x * uj.x - y.y * uj.y;
      acc.y += y.x * uj.y + y.y * uj.x;
    }
    const double2 sv = mul_conj(u[i], acc);  // S_i = u_i conj(I_i)
    const int tp = m.tpos[i], qi = m.qidx[i];
    if (tp >= 0) {
      const double ps = io.p_spec[s * m.n_theta + tp];
      fmx = nanmax(fmx, fabs(sv.x - ps));
      pspec += ps;
    } else {
      pslack += sv.x;
    }
    if (qi >= 0) fmx = nanmax(fmx, fabs(sv.y - io.q_spec[s * m.n_q + qi]));
  }
  double loss = 0.0;
  for (int b = t; b < m.n_br; b += kCertThreads) {
    const double2 uf = u[m.br_f[b]], ut = u[m.br_t[b]];
    const double2* y = m.br_y + 4 * (size_t)b;  // yff, yft, ytf, ytt
    const double2 ff = cmul(y[0], uf), ft = cmul(y[1], ut), tf = cmul(y[2], uf), tt = cmul(y[3], ut);
    const double2 i_f = make_double2(ff.x + ft.x, ff.y + ft.y);
    const double2 i_t = make_double2(tf.x + tt.x, tf.y + tt.y);
    loss += mul_conj(uf, i_f).x + mul_conj(ut, i_t).x;
  }
  fmx = block_max(fmx, red);
  pslack = block_sum(pslack, red);
  pspec = block_sum(pspec, red);
  loss = block_sum(loss, red);
  shunt = block_sum(shunt, red);
  if (t == 0) {
    if (io.mismatch_inf) io.mismatch_inf[s] = fmx;
    if (io.slack_balance) io.slack_balance[s] = pslack - ((loss + shunt) - pspec);
    if (io.branch_loss) io.branch_loss[s] = loss;
  }
}

__global__ void __launch_bounds__(kCertThreads) zb_kcl_kernel(ZbCertModel m, ZbCertIO io) {
  extern __shared__ __align__(16) unsigned char smem[];
  double2* v = reinterpret_cast<double2*>(smem);
  double2* r = v + m.n;
  double* red = reinterpret_cast<double*>(r + m.n);
  __shared__ int bad;
  const int64_t s = blockIdx.x;
  const int t = threadIdx.x;
  if (t == 0) bad = 0;
  for (int k = t; k < m.n; k += kCertThreads) v[k] = io.v[s * m.n + k];
  __syncthreads();
  for (int k = t; k < m.n; k += kCertThreads) {
    double2 acc = m.inj[k];  // Y_NS v_slack
    for (int e = m.rowptr[k]; e < m.rowptr[k + 1]; ++e) {
      const double2 y = m.val[e], vj = v[m.col[e]];
      acc.x += y.x * vj.x - y.y * vj.y;
      acc.y += y.x * vj.y + y.y * vj.x;
    }
    r[k] = acc;
  }
  __syncthreads();
  if (t == 0) {
    // r = i_net - i_loads, loads in the reference order (wye, then delta;
    // current_injection, distribution.py:573-610)
    for (int w = 0; w < m.n_wye; ++w) {
      const int p = m.wye_row[w];
      const double2 vp = v[p];
      if (hypot(vp.x, vp.y) <= m.floor) {
        bad = 1;
        break;
      }
      const double2 q = cdiv(io.s_wye[s * m.n_wye + w], vp);  // i_p += -conj(s / v_p)
      r[p].x += q.x;
      r[p].y -= q.y;
    }
    for (int d = 0; d < m.n_delta && !bad; ++d) {
      const int p = m.dp_row[d], q = m.dq_row[d];
      const double2 dv = make_double2(v[p].x - v[q].x, v[p].y - v[q].y);
      if (hypot(dv.x, dv.y) <= m.floor) {
        bad = 1;
        break;
      }
      const double2 c = cdiv(io.s_delta[s * m.n_delta + d], dv);  // i_line = conj(s / dv)
      r[p].x += c.x;  // i_p -= i_line
      r[p].y -= c.y;
      r[q].x -= c.x;  // i_q += i_line
      r[q].y += c.y;
    }
  }
  __syncthreads();
  double mx = 0.0;
  for (int k = t; k < m.n; k += kCertThreads) mx = nanmax(mx, hypot(r[k].x, r[k].y));
  mx = block_max(mx, red);
  if (t == 0) io.kcl[s] = bad ? __longlong_as_double(0x7ff0000000000000LL) : mx;
}

}  // namespace

size_t nr_cert_smem(int n_bus) { return (size_t)n_bus * sizeof(double2) + kCertThreads * sizeof(double); }

size_t zb_cert_smem(int n) { return (size_t)n * 2 * sizeof(double2) + kCertThreads * sizeof(double); }

cudaError_t launch_nr_cert(const NrCertModel& m, const NrCertIO& io, cudaStream_t st) {
  const size_t sm = nr_cert_smem(m.n_bus);
  cudaError_t e = cudaFuncSetAttribute(nr_cert_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  if (io.batch > 0) nr_cert_kernel<<<(unsigned)io.batch, kCertThreads, sm, st>>>(m, io);
  return cudaGetLastError();
}

cudaError_t launch_zb_kcl(const ZbCertModel& m, const ZbCertIO& io, cudaStream_t st) {
  const size_t sm = zb_cert_smem(m.n);
  cudaError_t e = cudaFuncSetAttribute(zb_kcl_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  if (io.batch > 0) zb_kcl_kernel<<<(unsigned)io.batch, kCertThreads, sm, st>>>(m, io);
  return cudaGetLastError();
}

}  // namespace acpf
