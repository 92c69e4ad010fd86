// The paper's Newton step on the GPU: matrix-free Jacobian-vector products
// and left-preconditioned restarted GMRES with the fast-decoupled (FD)
// preconditioner (an ablation of the exact
// sparse-LU step in nr_kernel.cu).
//
// Reference: `_newton_loop` (transmission.py:333-380) calling `gmres`
// (sparse.py:219-338) on `_jvp_operator` (transmission.py:218-236) with
// `apply_preconditioner` (transmission.py:292-298):
//   z_th = B'^-1 (r_th / V_th);  z_q = B''^-1 ((r_q - G z_th) / V_q)
// with B' = -Im Y[th,th] + eps I, B'' = -Im Y[q,q] + eps I, G = -Re Y[q,th]
// (network.py:519-543, transmission.py:259-266).
//
// Batched form: every vector is [rows][Bc] with the Bc scenarios of a chunk
// fastest, so per-row work is coalesced across scenarios and the two dense
// preconditioner solves of all scenarios are two GEMMs against the explicit
// inverses of the shared FD matrices, on the FP64 tensor cores (fd_gemm_kernel,
// DMMA). Each scenario runs its
// own GMRES (own Krylov basis, Hessenberg, Givens rotations, own iteration
// count and convergence), masked in lockstep kernels; dot products are
// fixed-order two-phase reductions, so results do not depend on the batch.

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "acpf_internal.cuh"

namespace acpf {

namespace {

constexpr int kT = 256;
constexpr int kDotChunk = 64;  // rows per partial dot product

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

unsigned blocks_for(int64_t n) { return (unsigned)((n + kT - 1) / kT); }

// ---- FD solves: C[M][N] = A[M][K] B[K][N] (row-major, FP64) on DMMA ----
// A = (B' + eps I)^-1 or (B'' + eps I)^-1 (shared by every scenario), B the
// chunk's scaled residuals [rows][Bc]. CTA tile BM x BN, K steps of 16
// through a 3-stage cp.async ring; warps of WM x WN mma.m8n8k4 accumulator
// tiles. Small CTAs (64 x 64, 4 warps of 32 x 32) so that several are
// resident per SM: their independent DMMA streams keep the FP64 tensor pipe
// busy and the grid splits into many short waves. Shared rows are padded
// (A BK+4, B BN+4 doubles) so the fragment loads of a half-warp hit 16
// distinct 8-byte bank pairs. Edges are zero-filled (cp.async src-size 0),
// so any M, N, K and unaligned leading dimensions work. Each output element
// is one fixed-order sum, independent of the batch and of the grid.
constexpr int kGBK = 16, kGStages = 3;

__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool pred) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(pred ? 8 : 0)
               : "memory");
}

template <int BM, int BN, int WM, int WN>
struct GemmCfg {
  static constexpr int kWarpsN = BN / (8 * WN);
  static constexpr int kThreads = 32 * (BM / (8 * WM)) * kWarpsN;
  static constexpr int kLdA = kGBK + 4, kLdB = BN + 4;
  static constexpr int kStageA = BM * kLdA, kStageB = kGBK * kLdB;
  static constexpr size_t kSmem = (size_t)kGStages * (kStageA + kStageB) * sizeof(double);
};

template <int BM, int BN, int WM, int WN>
__global__ void __launch_bounds__(GemmCfg<BM, BN, WM, WN>::kThreads, GemmCfg<BM, BN, WM, WN>::kThreads <= 128 ? 4 : 1)
    fd_gemm_kernel(int M, int N, int K, const double* __restrict__ A, int lda, const double* __restrict__ B,
                   int ldb, double* __restrict__ C, int ldc) {
  using G = GemmCfg<BM, BN, WM, WN>;
  constexpr int T = G::kThreads;
  extern __shared__ __align__(16) double gsm[];
  double* const As = gsm;
  double* const Bs = gsm + kGStages * G::kStageA;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / G::kWarpsN, wn = warp % G::kWarpsN;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int nk = (K + kGBK - 1) / kGBK;
  auto load = [&](int stage, int kt) {
    const int k0 = kt * kGBK;
    double* const as = As + stage * G::kStageA;
    double* const bs = Bs + stage * G::kStageB;
#pragma unroll
    for (int i = 0; i < BM * kGBK / T; ++i) {
      const int e = tid + T * i, r = e / kGBK, c = e % kGBK;
      const bool ok = m0 + r < M && k0 + c < K;
      cp_async8(as + r * G::kLdA + c, ok ? A + (size_t)(m0 + r) * lda + k0 + c : A, ok);
    }
#pragma unroll
    for (int i = 0; i < kGBK * BN / T; ++i) {
      const int e = tid + T * i, r = e / BN, c = e % BN;
      const bool ok = k0 + r < K && n0 + c < N;
      cp_async8(bs + r * G::kLdB + c, ok ? B + (size_t)(k0 + r) * ldb + n0 + c : B, ok);
    }
  };
  double acc[WM][WN][2];
#pragma unroll
  for (int i = 0; i < WM; ++i)
#pragma unroll
    for (int j = 0; j < WN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
  for (int s = 0; s < kGStages - 1; ++s) {
    if (s < nk) load(s, s);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  const int ar = wm * 8 * WM + (lane >> 2), ac = lane & 3;      // A fragment: row, k
  const int br = lane & 3, bcol = wn * 8 * WN + (lane >> 2);   // B fragment: k, column
  for (int kt = 0; kt < nk; ++kt) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(kGStages - 2) : "memory");
    __syncthreads();
    if (kt + kGStages - 1 < nk) load((kt + kGStages - 1) % kGStages, kt + kGStages - 1);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    const double* const as = As + (kt % kGStages) * G::kStageA;
    const double* const bs = Bs + (kt % kGStages) * G::kStageB;
#pragma unroll
    for (int kk = 0; kk < kGBK; kk += 4) {
      double a[WM], b[WN];
#pragma unroll
      for (int i = 0; i < WM; ++i) a[i] = as[(ar + 8 * i) * G::kLdA + kk + ac];
#pragma unroll
      for (int j = 0; j < WN; ++j) b[j] = bs[(kk + br) * G::kLdB + bcol + 8 * j];
#pragma unroll
      for (int i = 0; i < WM; ++i)
#pragma unroll
        for (int j = 0; j < WN; ++j)
          asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
              : "+d"(acc[i][j][0]), "+d"(acc[i][j][1])
              : "d"(a[i]), "d"(b[j]));
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  const int cr = m0 + wm * 8 * WM + (lane >> 2), cc = n0 + wn * 8 * WN + 2 * (lane & 3);
#pragma unroll
  for (int i = 0; i < WM; ++i) {
    const int r = cr + 8 * i;
    if (r >= M) continue;
#pragma unroll
    for (int j = 0; j < WN; ++j) {
      const int c = cc + 8 * j;
      double* const dst = C + (size_t)r * ldc + c;
      if (c + 1 < N && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
        *reinterpret_cast<double2*>(dst) = make_double2(acc[i][j][0], acc[i][j][1]);
      } else {
        if (c < N) dst[0] = acc[i][j][0];
        if (c + 1 < N) dst[1] = acc[i][j][1];
      }
    }
  }
}

template <int BM, int BN, int WM, int WN>
cudaError_t fd_gemm_launch(int M, int N, int K, const double* A, int lda, const double* B, int ldb, double* C,
                           int ldc, cudaStream_t st) {
  using G = GemmCfg<BM, BN, WM, WN>;
  // per call, not cached: the attribute belongs to the current device's context
  const cudaError_t attr = cudaFuncSetAttribute(fd_gemm_kernel<BM, BN, WM, WN>,
                                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::kSmem);
  if (attr != cudaSuccess) return attr;
  const dim3 grid((unsigned)((N + BN - 1) / BN), (unsigned)((M + BM - 1) / BM));
  fd_gemm_kernel<BM, BN, WM, WN><<<grid, G::kThreads, G::kSmem, st>>>(M, N, K, A, lda, B, ldb, C, ldc);
  return cudaGetLastError();
}

// ACPF_FD_GEMM_TILE: 0 (default) 64 x 64 CTAs of 4 warps; 1 128 x 128 of 8 warps
cudaError_t fd_gemm(int M, int N, int K, const double* A, int lda, const double* B, int ldb, double* C, int ldc,
                    cudaStream_t st) {
  static const int tile = [] {
    const char* v = std::getenv("ACPF_FD_GEMM_TILE");
    return v ? std::atoi(v) : 0;
  }();
  if (tile == 1) return fd_gemm_launch<128, 128, 8, 4>(M, N, K, A, lda, B, ldb, C, ldc, st);
  return fd_gemm_launch<64, 64, 4, 4>(M, N, K, A, lda, B, ldb, C, ldc, st);
}

// ---- state: u = V e^{j th}, phase = e^{j th}, I = Y u; mismatch F packed
// [th block: P - p_spec; q block: Q - q_spec]; ||F||inf and flags per scenario
__global__ void gm_phasor(GmModel m, GmWork w) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)m.n_bus * w.bc) return;
  const int s = (int)(t % w.bc);  // [bus][scenario] layout: t = bus * Bc + s
  if (!w.nactive[s]) return;
  const double th = w.th[t], v = w.vm[t];
  double sn, cs;
  sincos(th, &sn, &cs);
  w.ph[t] = make_double2(cs, sn);
  w.u[t] = make_double2(v * cs, v * sn);
  if (v <= 0.0) atomicOr(&w.flags[s], 4);
}

__global__ void gm_mismatch(GmModel m, GmWork w) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)m.n_bus * w.bc) return;
  const int i = (int)(t / w.bc), s = (int)(t % w.bc);
  if (!w.nactive[s]) return;
  double2 acc = make_double2(0.0, 0.0);
  for (int e = m.y_rowptr[i]; e < m.y_rowptr[i + 1]; ++e) {
    const double2 y = m.y_val[e], uj = w.u[(size_t)m.y_col[e] * w.bc + s];
    acc.x += y.x * uj.x - y.y * uj.y;
    acc.y += y.x * uj.y + y.y * uj.x;
  }
  w.ic[t] = make_double2(acc.x, -acc.y);  // conj(I)
  const double2 u = w.u[t];
  const double p = u.x * acc.x + u.y * acc.y, q = u.y * acc.x - u.x * acc.y;  // S = u conj(I)
  double fm = 0.0;
  int bad = 0;
  const int tp = m.tpos[i], qi = m.qidx[i];
  if (tp >= 0) {
    const double f = p - w.p_spec[(size_t)s * m.n_theta + tp];
    w.b[(size_t)tp * w.bc + s] = -f;  // GMRES right-hand side -F
    bad |= isnan(f) ? 1 : (isinf(f) ? 2 : 0);
    fm = fabs(f);
  }
  if (qi >= 0) {
    const double f = q - w.q_spec[(size_t)s * m.n_q + qi];
    w.b[(size_t)(m.n_theta + qi) * w.bc + s] = -f;
    bad |= isnan(f) ? 1 : (isinf(f) ? 2 : 0);
    fm = fm < fabs(f) ? fabs(f) : fm;
  }
  if (fm > 0.0) atomicMax(&w.fmax_bits[s], (unsigned long long)__double_as_longlong(fm));
  if (bad) atomicOr(&w.flags[s], bad);
}

// the reference exit checks in order (transmission.py:347-359)
__global__ void gm_check(GmWork w, int k, int max_newton, double tol) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= w.bc) return;
  bool act = w.nactive[s];
  if (act) {
    const double fmx = __longlong_as_double((long long)w.fmax_bits[s]);
    const int fl = w.flags[s];
    int st = -1;
    double fo = fmx;
    if (fl & 3) {
      st = ACPF_NR_NONFINITE;
      fo = (fl & 1) ? __longlong_as_double(0x7ff8000000000000LL) : __longlong_as_double(0x7ff0000000000000LL);
    } else if (fmx <= tol) {
      st = ACPF_NR_CONVERGED;
    } else if (fl & 4) {
      st = ACPF_NR_VMAG_LE0;
    } else if (k == max_newton) {
      st = ACPF_NR_MAX_ITER;
    }
    w.fout[s] = fo;
    if (st >= 0) {
      w.status[s] = st;
      w.iters[s] = st == ACPF_NR_MAX_ITER ? max_newton : k;
      w.nactive[s] = 0;
      act = false;
    }
  }
  w.fmax_bits[s] = 0ull;
  w.flags[s] = 0;
  w.gstate[s] = act ? 1 : 0;  // 1: GMRES running for this scenario
  if (act) atomicAdd(w.count, 1);
}

// ---- operator: out = J(x) v  (_jvp_operator): du = phase dV + j u dth;
// ds = du conj(I) + u conj(Y du); out = [Re ds over th block; Im ds over q block]
__global__ void gm_jvp_du(GmModel m, GmWork w, const double* v, const int* mask) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)m.n_bus * w.bc) return;
  const int i = (int)(t / w.bc), s = (int)(t % w.bc);
  if (!mask[s]) return;
  const int tp = m.tpos[i], qi = m.qidx[i];
  const double dth = tp >= 0 ? v[(size_t)tp * w.bc + s] : 0.0;
  const double dvm = qi >= 0 ? v[(size_t)(m.n_theta + qi) * w.bc + s] : 0.0;
  const double2 ph = w.ph[t], u = w.u[t];
  w.du[t] = make_double2(ph.x * dvm - u.y * dth, ph.y * dvm + u.x * dth);
}

__global__ void gm_jvp_ds(GmModel m, GmWork w, double* out, const int* mask) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)m.n_bus * w.bc) return;
  const int i = (int)(t / w.bc), s = (int)(t % w.bc);
  if (!mask[s]) return;
  const int tp = m.tpos[i], qi = m.qidx[i];
  if (tp < 0 && qi < 0) return;
  double2 acc = make_double2(0.0, 0.0);
  for (int e = m.y_rowptr[i]; e < m.y_rowptr[i + 1]; ++e) {
    const double2 y = m.y_val[e], d = w.du[(size_t)m.y_col[e] * w.bc + s];
    acc.x += y.x * d.x - y.y * d.y;
    acc.y += y.x * d.y + y.y * d.x;
  }
  const double2 a = cmul(w.du[t], w.ic[t]);
  const double2 u = w.u[t];
  const double2 b = make_double2(u.x * acc.x + u.y * acc.y, u.y * acc.x - u.x * acc.y);  // u conj(Y du)
  if (tp >= 0) out[(size_t)tp * w.bc + s] = a.x + b.x;
  if (qi >= 0) out[(size_t)(m.n_theta + qi) * w.bc + s] = a.y + b.y;
}

// ---- FD preconditioner pieces
__global__ void gm_scale_th(GmModel m, GmWork w, const double* in, double* out, const int* mask) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)m.n_theta * w.bc) return;
  const int k = (int)(t / w.bc), s = (int)(t % w.bc);
  out[t] = mask[s] ? in[t] / w.vm[(size_t)m.theta_block[k] * w.bc + s] : 0.0;
}

__global__ void gm_couple_q(GmModel m, GmWork w, const double* in, const double* zth, double* out,
                            const int* mask) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)m.n_q * w.bc) return;
  const int k = (int)(t / w.bc), s = (int)(t % w.bc);
  if (!mask[s]) {
    out[t] = 0.0;
    return;
  }
  double acc = 0.0;
  for (int e = m.g_rowptr[k]; e < m.g_rowptr[k + 1]; ++e) acc += m.g_val[e] * zth[(size_t)m.g_col[e] * w.bc + s];
  out[t] = (in[(size_t)(m.n_theta + k) * w.bc + s] - acc) / w.vm[(size_t)m.q_block[k] * w.bc + s];
}

__global__ void gm_copy(int64_t n, const double* in, double* out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) out[t] = in[t];
}

// ---- per-scenario dot products over nJ rows: partial sums of kDotChunk
// rows, then a fixed-order sum
__global__ void gm_dot_partial(int nj, int bc, const double* a, const double* b, double* part, const int* mask) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  const int c = blockIdx.y;
  if (s >= bc || !mask[s]) return;
  const int r0 = c * kDotChunk, r1 = min(nj, r0 + kDotChunk);
  double acc = 0.0;
  for (int r = r0; r < r1; ++r) acc += a[(size_t)r * bc + s] * b[(size_t)r * bc + s];
  part[(size_t)c * bc + s] = acc;
}

__global__ void gm_dot_final(int nchunk, int bc, const double* part, double* out, const int* mask) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= bc || !mask[s]) return;
  double acc = 0.0;
  for (int c = 0; c < nchunk; ++c) acc += part[(size_t)c * bc + s];
  out[s] = acc;
}

// w -= h v (h per scenario)
__global__ void gm_axpy(int64_t n, int bc, const double* h, const double* v, double* wv, const int* mask) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int s = (int)(t % bc);
  if (mask[s]) wv[t] -= h[s] * v[t];
}

// out = in / d (d per scenario)
__global__ void gm_div(int64_t n, int bc, const double* in, const double* d, double* out, const int* mask) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int s = (int)(t % bc);
  if (mask[s]) out[t] = in[t] / d[s];
}

// beta0 = ||M^-1 b||; scenarios with beta0 == 0 finish with dx = 0
__global__ void gm_begin(GmWork w) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= w.bc || !w.gstate[s]) return;
  const double b0 = sqrt(w.scal[s]);
  w.beta0[s] = b0;
  w.gsum[s] = 0;
  if (b0 == 0.0) w.gstate[s] = 0;
}

// restart boundary: beta = ||r||; relres check; starts a cycle (cycle_on) if
// the scenario must continue
__global__ void gm_cycle_start(GmWork w, int cycle, int max_outer, double tol) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= w.bc) return;
  w.cyc[s] = 0;
  if (w.gstate[s] != 1) return;
  const double beta = cycle == 0 ? w.beta0[s] : sqrt(w.scal[s]);
  const double rel = beta / w.beta0[s];
  w.relres[s] = rel;
  if (rel <= tol) {
    w.gstate[s] = 0;  // converged
    return;
  }
  if (cycle == max_outer || w.brk[s]) {
    w.gstate[s] = 2;  // stagnated / breakdown: keep x, stop
    return;
  }
  w.g[s] = beta;  // g[0]
  w.beta[s] = beta;
  w.kk[s] = 0;
  w.cyc[s] = 1;
  atomicAdd(w.count, 1);
}

// Arnoldi column j: h[j+1, j] = ||w||, rotations, residual estimate and the
// stop tests of the reference inner loop
__global__ void gm_givens(GmWork w, int j, int m, double tol) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= w.bc || !w.cyc[s]) return;
  const int bc = w.bc;
  auto H = [&](int r, int c) -> double& { return w.h[((size_t)r * m + c) * bc + s]; };
  const double hnorm = sqrt(w.scal[s]);
  H(j + 1, j) = hnorm;
  for (int i = 0; i < j; ++i) {
    const double c = w.cs[(size_t)i * bc + s], sn = w.sn[(size_t)i * bc + s];
    const double t = c * H(i, j) + sn * H(i + 1, j);
    H(i + 1, j) = -sn * H(i, j) + c * H(i + 1, j);
    H(i, j) = t;
  }
  const double denom = hypot(H(j, j), H(j + 1, j));
  if (denom == 0.0) {  // hard breakdown: column contributed nothing
    w.brk[s] = 1;
    w.kk[s] = j;
    w.cyc[s] = 0;
    return;
  }
  const double c = H(j, j) / denom, sn = H(j + 1, j) / denom;
  w.cs[(size_t)j * bc + s] = c;
  w.sn[(size_t)j * bc + s] = sn;
  H(j, j) = denom;
  H(j + 1, j) = 0.0;
  const double gj = w.g[(size_t)j * bc + s];
  w.g[(size_t)(j + 1) * bc + s] = -sn * gj;
  w.g[(size_t)j * bc + s] = c * gj;
  w.gsum[s] += 1;
  w.kk[s] = j + 1;
  const double rel = fabs(w.g[(size_t)(j + 1) * bc + s]) / w.beta0[s];
  if (hnorm <= 1e-14 * w.beta0[s]) {
    if (rel > tol) w.brk[s] = 1;
    w.cyc[s] = 0;
    return;
  }
  if (rel <= tol || j + 1 == m) {
    w.cyc[s] = 0;
    return;
  }
  w.scal[s] = hnorm;  // v[j+1] = w / hnorm
  atomicAdd(w.count, 1);
}

// y = H[:k,:k]^-1 g[:k] by back substitution (per scenario)
__global__ void gm_backsolve(GmWork w, int m) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= w.bc || w.kk[s] == 0) return;
  const int bc = w.bc, k = w.kk[s];
  for (int i = k - 1; i >= 0; --i) {
    double acc = 0.0;
    for (int c = i + 1; c < k; ++c) acc += w.h[((size_t)i * m + c) * bc + s] * w.y[(size_t)c * bc + s];
    w.y[(size_t)i * bc + s] = (w.g[(size_t)i * bc + s] - acc) / w.h[((size_t)i * m + i) * bc + s];
  }
}

// x += V[:k]^T y
__global__ void gm_xupdate(int nj, int bc, const double* vb, const double* y, const int* kk, double* x) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)nj * bc) return;
  const int s = (int)(t % bc);
  const int k = kk[s];
  double acc = 0.0;
  for (int i = 0; i < k; ++i) acc += vb[(size_t)i * nj * bc + t] * y[(size_t)i * bc + s];
  if (k) x[t] += acc;
}

// r = b - A x (in place on ax)
__global__ void gm_resid(int64_t n, int bc, const double* b, double* ax, const int* mask) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  if (mask[t % bc]) ax[t] = b[t] - ax[t];
}

// state += dx (transmission.py:378)
__global__ void gm_apply(GmModel m, GmWork w) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)m.nj * w.bc) return;
  const int k = (int)(t / w.bc), s = (int)(t % w.bc);
  if (!w.nactive[s]) return;
  if (k < m.n_theta)
    w.th[(size_t)m.theta_block[k] * w.bc + s] += w.x[t];
  else
    w.vm[(size_t)m.q_block[k - m.n_theta] * w.bc + s] += w.x[t];
}

__global__ void gm_init(GmModel m, GmWork w, int64_t nb) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)m.n_bus * w.bc) return;
  const int i = (int)(t / w.bc), s = (int)(t % w.bc);
  w.th[t] = m.theta_init[i];
  w.vm[t] = m.vmag_init[i];
  if (i == 0) {
    w.nactive[s] = s < nb;
    w.status[s] = 0;
    w.iters[s] = 0;
    w.fout[s] = 0.0;
    w.fmax_bits[s] = 0ull;
    w.flags[s] = 0;
    w.gtotal[s] = 0;
    w.gdiag[s] = 0;
    w.gdiag_k[s] = -1;
    w.gdiag_rel[s] = 0.0;
  }
}

// per Newton step: GMRES totals and the first diagnostic (1 breakdown, 2 stagnation)
__global__ void gm_step_end(GmWork w, int k) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= w.bc || !w.nactive[s]) return;
  w.gtotal[s] += w.gsum[s];
  w.gsteps[(size_t)k * w.bc + s] = w.gsum[s];
  // transmission.py:371-376: a breakdown always (re)sets the diagnostic, a
  // stagnation only when none is set yet
  if (w.brk[s]) {
    w.gdiag[s] = 1;
    w.gdiag_k[s] = k;
  } else if (w.gstate[s] == 2 && w.gdiag[s] == 0) {
    w.gdiag[s] = 2;
    w.gdiag_k[s] = k;
    w.gdiag_rel[s] = w.relres[s];
  }
}

__global__ void gm_output(GmModel m, GmWork w, int64_t nb, int max_newton, double* theta_out, double* vmag_out,
                          uint8_t* converged, int32_t* iterations, double* fnorm, int32_t* status,
                          int32_t* gmres_steps, int32_t* gmres_diag, int32_t* gmres_diag_k,
                          double* gmres_diag_relres) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)m.n_bus * w.bc) return;
  const int i = (int)(t / w.bc), s = (int)(t % w.bc);
  if (s >= nb) return;
  theta_out[(size_t)s * m.n_bus + i] = w.th[t];
  vmag_out[(size_t)s * m.n_bus + i] = w.vm[t];
  if (i == 0) {
    const int st = w.status[s];
    if (converged) converged[s] = st == ACPF_NR_CONVERGED;
    if (iterations) iterations[s] = w.iters[s];
    if (fnorm) fnorm[s] = w.fout[s];
    if (status) status[s] = st;
    if (gmres_steps)
      for (int k = 0; k < max_newton; ++k)
        gmres_steps[(size_t)s * max_newton + k] = k < w.iters[s] ? w.gsteps[(size_t)k * w.bc + s] : 0;
    if (gmres_diag) gmres_diag[s] = w.gdiag[s];
    if (gmres_diag_k) gmres_diag_k[s] = w.gdiag_k[s];
    if (gmres_diag_relres) gmres_diag_relres[s] = w.gdiag_rel[s];
  }
}

}  // namespace

size_t gmres_work_doubles(const GmModel& m, int bc, int restart) {
  const size_t nj = m.nj, nb = m.n_bus, B = bc, mm = restart;
  return B * (2 * nb            // th, vm
              + 8 * nb          // u, ph, ic, du (complex)
              + 5 * nj          // b, x, wv, t1, t2
              + (mm + 1) * nj   // Krylov basis
              + (mm + 1) * mm   // Hessenberg
              + 2 * mm          // cs, sn
              + 2 * (mm + 1)    // g, y
              + ((nj + kDotChunk - 1) / kDotChunk)  // dot partials
              + 8);             // scalars
}

cudaError_t gmres_output(const GmModel& m, const GmWork& w, int64_t nb, int max_newton, double* theta_out,
                         double* vmag_out, uint8_t* converged, int32_t* iterations, double* fnorm,
                         int32_t* status, int32_t* gmres_steps, int32_t* gmres_diag, int32_t* gmres_diag_k,
                         double* gmres_diag_relres, cudaStream_t st) {
  gm_output<<<blocks_for((int64_t)m.n_bus * w.bc), kT, 0, st>>>(m, w, nb, max_newton, theta_out, vmag_out,
                                                                 converged, iterations, fnorm, status, gmres_steps,
                                                                 gmres_diag, gmres_diag_k, gmres_diag_relres);
  return cudaGetLastError();
}

// The whole GMRES-Newton solve of one chunk (host loop; one 4-byte D2H per
// Newton step and per GMRES iteration for the active counts).
cudaError_t gmres_newton(const GmModel& m, GmWork& w, int64_t nb, double tol, int max_newton,
                         double gtol, int restart, int max_outer, bool fd, cudaStream_t st) {
  const int bc = w.bc, nj = m.nj, mm = restart;
  const int64_t nbus_b = (int64_t)m.n_bus * bc, nj_b = (int64_t)nj * bc;
  const int nchunk = (nj + kDotChunk - 1) / kDotChunk;
  const unsigned sb = blocks_for(bc);
  cudaError_t e;
  auto count = [&](int& out) -> cudaError_t {
    cudaError_t r = cudaMemcpyAsync(w.host_count, w.count, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (r == cudaSuccess) r = cudaStreamSynchronize(st);
    out = *w.host_count;
    return r;
  };
  auto zero_count = [&]() { return cudaMemsetAsync(w.count, 0, sizeof(int), st); };
  auto dot = [&](const double* a, const double* b, const int* mask, double* out) {
    gm_dot_partial<<<dim3(sb, nchunk), kT, 0, st>>>(nj, bc, a, b, w.part, mask);
    gm_dot_final<<<sb, kT, 0, st>>>(nchunk, bc, w.part, out, mask);
  };
  // out = M^-1 A v (or M^-1 v when op == false)
  auto precond = [&](const double* in, double* out, const int* mask) -> cudaError_t {
    if (!fd) {
      gm_copy<<<blocks_for(nj_b), kT, 0, st>>>(nj_b, in, out);
      return cudaGetLastError();
    }
    gm_scale_th<<<blocks_for((int64_t)m.n_theta * bc), kT, 0, st>>>(m, w, in, w.t2, mask);
    // z_th[n_theta][Bc] = B'^-1 t, z_q = B''^-1 ((r_q - G z_th) / V_q)
    cudaError_t r = cudaSuccess;
    if (m.n_theta) r = fd_gemm(m.n_theta, bc, m.n_theta, m.binv1, m.n_theta, w.t2, bc, out, bc, st);
    if (r == cudaSuccess && m.n_q) {
      gm_couple_q<<<blocks_for((int64_t)m.n_q * bc), kT, 0, st>>>(m, w, in, out, w.t2, mask);
      r = fd_gemm(m.n_q, bc, m.n_q, m.binv2, m.n_q, w.t2, bc, out + (size_t)m.n_theta * bc, bc, st);
    }
    return r == cudaSuccess ? cudaGetLastError() : r;
  };
  auto op = [&](const double* v, double* out, const int* mask) {
    gm_jvp_du<<<blocks_for(nbus_b), kT, 0, st>>>(m, w, v, mask);
    gm_jvp_ds<<<blocks_for(nbus_b), kT, 0, st>>>(m, w, out, mask);
  };

  gm_init<<<blocks_for(nbus_b), kT, 0, st>>>(m, w, nb);
  for (int k = 0; k <= max_newton; ++k) {
    gm_phasor<<<blocks_for(nbus_b), kT, 0, st>>>(m, w);
    gm_mismatch<<<blocks_for(nbus_b), kT, 0, st>>>(m, w);
    if ((e = zero_count()) != cudaSuccess) return e;
    gm_check<<<sb, kT, 0, st>>>(w, k, max_newton, tol);
    int act = 0;
    if ((e = count(act)) != cudaSuccess) return e;
    if (act == 0) break;
    // GMRES on J dx = -F from x = 0 (sparse.py:219-338)
    if ((e = cudaMemsetAsync(w.x, 0, nj_b * sizeof(double), st)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(w.brk, 0, bc * sizeof(int), st)) != cudaSuccess) return e;
    if ((e = precond(w.b, w.vb, w.gstate)) != cudaSuccess) return e;  // r0 = M^-1 b
    dot(w.vb, w.vb, w.gstate, w.scal);
    gm_begin<<<sb, kT, 0, st>>>(w);
    for (int cycle = 0; cycle <= max_outer; ++cycle) {
      if (cycle > 0) {  // true preconditioned residual at the restart boundary
        op(w.x, w.t1, w.gstate);
        gm_resid<<<blocks_for(nj_b), kT, 0, st>>>(nj_b, bc, w.b, w.t1, w.gstate);
        if ((e = precond(w.t1, w.vb, w.gstate)) != cudaSuccess) return e;
        dot(w.vb, w.vb, w.gstate, w.scal);
      }
      if ((e = zero_count()) != cudaSuccess) return e;
      gm_cycle_start<<<sb, kT, 0, st>>>(w, cycle, max_outer, gtol);
      int running = 0;
      if ((e = count(running)) != cudaSuccess) return e;
      if (running == 0) break;
      gm_div<<<blocks_for(nj_b), kT, 0, st>>>(nj_b, bc, w.vb, w.beta, w.vb, w.cyc);  // v0 = r / beta
      for (int j = 0; j < mm; ++j) {
        double* vj = w.vb + (size_t)j * nj_b;
        op(vj, w.t1, w.cyc);
        if ((e = precond(w.t1, w.wv, w.cyc)) != cudaSuccess) return e;
        for (int i = 0; i <= j; ++i) {  // modified Gram-Schmidt, fixed order
          double* vi = w.vb + (size_t)i * nj_b;
          double* hij = w.h + ((size_t)i * mm + j) * bc;
          dot(vi, w.wv, w.cyc, hij);
          gm_axpy<<<blocks_for(nj_b), kT, 0, st>>>(nj_b, bc, hij, vi, w.wv, w.cyc);
        }
        dot(w.wv, w.wv, w.cyc, w.scal);
        if ((e = zero_count()) != cudaSuccess) return e;
        gm_givens<<<sb, kT, 0, st>>>(w, j, mm, gtol);
        int cont = 0;
        if ((e = count(cont)) != cudaSuccess) return e;
        if (cont == 0) break;
        gm_div<<<blocks_for(nj_b), kT, 0, st>>>(nj_b, bc, w.wv, w.scal, w.vb + (size_t)(j + 1) * nj_b, w.cyc);
      }
      gm_backsolve<<<sb, kT, 0, st>>>(w, mm);
      gm_xupdate<<<blocks_for(nj_b), kT, 0, st>>>(nj, bc, w.vb, w.y, w.kk, w.x);
      if ((e = cudaMemsetAsync(w.kk, 0, bc * sizeof(int), st)) != cudaSuccess) return e;
    }
    gm_step_end<<<sb, kT, 0, st>>>(w, k);
    gm_apply<<<blocks_for(nj_b), kT, 0, st>>>(m, w);
  }
  return cudaGetLastError();
}

}  // namespace acpf
