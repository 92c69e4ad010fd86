// Z-Bus network reduction on the device.
//
// Reference `reduce_zbus` (distribution.py:431-517) factors the dense
// non-slack block Y_NN with LAPACK getrf on the host and solves for
// v0 = -Y_NN^-1 Y_NS v_slack; this engine additionally needs the load
// columns Z[:, l] = Y_NN^-1 E_l. Here Y_NN (CSR from the host model) is
// scattered into a dense column-major matrix on the device, factored with
// cuSOLVER getrf (partial pivoting, as LAPACK) and both right-hand-side sets
// are solved by lu_solve_columns (one CTA per column; cuSOLVER getrs took
// ~0.4 s for these 56 columns). The reference's singularity test (non-finite LU or
// min |U_ii| <= n eps max|Y|) is applied to the device factor.

#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "acpf_internal.cuh"

namespace acpf {

namespace {

__global__ void scatter_csr_colmajor(int n, const int32_t* rowptr, const int32_t* col, const double2* val,
                                     double2* a) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  for (int e = rowptr[r]; e < rowptr[r + 1]; ++e) {
    double2* p = a + (size_t)col[e] * n + r;
    *p = make_double2(p->x + val[e].x, p->y + val[e].y);  // duplicates sum, like scipy
  }
}

__global__ void fill_rhs(int n, int n_l, const int32_t* l_index, const double2* rhs0, double2* b) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t total = (size_t)n * (n_l + 1);
  if (i >= total) return;
  const int c = (int)(i / n), r = (int)(i % n);
  b[i] = c < n_l ? make_double2(l_index[c] == r ? 1.0 : 0.0, 0.0) : rhs0[r];
}

// min |U_ii| and a non-finite flag over the factor (one block)
__global__ void diag_check(int n, const double2* a, double* min_abs, int* nonfinite) {
  __shared__ double red[256];
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  double m = INFINITY;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double2 d = a[(size_t)i * n + i];
    const double v = hypot(d.x, d.y);
    if (!isfinite(d.x) || !isfinite(d.y)) bad = 1;
    m = fmin(m, v);
  }
  red[threadIdx.x] = m;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = fmin(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *min_abs = red[0];
    *nonfinite = bad;
  }
}

__global__ void any_nonfinite(size_t count, const double2* a, int* flag) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count && (!isfinite(a[i].x) || !isfinite(a[i].y))) *flag = 1;
}

// Solve LU x = P b for each right-hand side column (one CTA per column, the
// column staged in shared memory): the row interchanges of getrf (1-based
// ipiv, applied in order as LAPACK getrs does), then unit-lower forward and
// upper back substitution, one pivot step per barrier. The factor is read
// column by column (coalesced) from L2.
__global__ void __launch_bounds__(1024) lu_solve_columns(int n, const double2* __restrict__ a,
                                                         const int* __restrict__ ipiv, double2* b) {
  extern __shared__ double2 x[];
  double2* col = b + (size_t)blockIdx.x * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) x[i] = col[i];
  __syncthreads();
  if (threadIdx.x == 0)
    for (int i = 0; i < n; ++i) {
      const int pi = ipiv[i] - 1;
      if (pi != i) {
        const double2 t = x[i];
        x[i] = x[pi];
        x[pi] = t;
      }
    }
  __syncthreads();
  for (int j = 0; j < n; ++j) {  // L y = P b (unit diagonal)
    const double2 xj = x[j];
    const double2* lj = a + (size_t)j * n;
    for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) {
      const double2 l = lj[i];
      x[i].x -= l.x * xj.x - l.y * xj.y;
      x[i].y -= l.x * xj.y + l.y * xj.x;
    }
    __syncthreads();
  }
  for (int j = n - 1; j >= 0; --j) {  // U x = y
    const double2* uj = a + (size_t)j * n;
    if (threadIdx.x == 0) {
      const double2 u = uj[j], v = x[j];
      double2 q;
      if (fabs(u.x) >= fabs(u.y)) {
        const double r = u.y / u.x, d = u.x + u.y * r;
        q = make_double2((v.x + v.y * r) / d, (v.y - v.x * r) / d);
      } else {
        const double r = u.x / u.y, d = u.x * r + u.y;
        q = make_double2((v.x * r + v.y) / d, (v.y * r - v.x) / d);
      }
      x[j] = q;
    }
    __syncthreads();
    const double2 xj = x[j];
    for (int i = threadIdx.x; i < j; i += blockDim.x) {
      const double2 u = uj[i];
      x[i].x -= u.x * xj.x - u.y * xj.y;
      x[i].y -= u.x * xj.y + u.y * xj.x;
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) col[i] = x[i];
}

}  // namespace

acpf_status zbus_reduce_device(int device, int n, const int32_t* rowptr, const int32_t* col, const double* val,
                               const double* rhs0, int n_l, const int32_t* l_index, double* zl_out,
                               double* v0_out, double* min_pivot_out) {
  cudaSetDevice(device);
  const bool dbg = std::getenv("ACPF_DEBUG_REDUCE") != nullptr;
  auto t0 = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!dbg) return;
    cudaDeviceSynchronize();
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    std::fprintf(stderr, "[acpf_zbus_reduce] %-10s %8.2f ms\n", what, ms);
  };
  const int64_t nnz = rowptr[n];
  std::vector<void*> ptrs;
  auto cleanup = [&]() {
    for (void* q : ptrs) cudaFree(q);
  };
  auto alloc = [&](size_t bytes) -> void* {
    void* q = nullptr;
    if (cudaMalloc(&q, bytes ? bytes : 1) != cudaSuccess) return nullptr;
    ptrs.push_back(q);
    return q;
  };
  const size_t nn = (size_t)n * n, nr = (size_t)n * (n_l + 1);
  double2* a = (double2*)alloc(nn * sizeof(double2));
  double2* b = (double2*)alloc(nr * sizeof(double2));
  int32_t* d_rp = (int32_t*)alloc((size_t)(n + 1) * 4);
  int32_t* d_col = (int32_t*)alloc((size_t)nnz * 4);
  double2* d_val = (double2*)alloc((size_t)nnz * sizeof(double2));
  double2* d_rhs0 = (double2*)alloc((size_t)n * sizeof(double2));
  int32_t* d_l = (int32_t*)alloc((size_t)n_l * 4);
  int* ipiv = (int*)alloc((size_t)n * sizeof(int));
  int* info = (int*)alloc(2 * sizeof(int));
  double* d_min = (double*)alloc(sizeof(double));
  if (!a || !b || !d_rp || !d_col || !d_val || !d_rhs0 || !d_l || !ipiv || !info || !d_min) {
    cleanup();
    set_error("acpf_zbus_reduce: device allocation failed");
    return ACPF_ENOMEM;
  }
  cudaError_t e = cudaMemset(a, 0, nn * sizeof(double2));
  if (e == cudaSuccess) e = cudaMemcpy(d_rp, rowptr, (size_t)(n + 1) * 4, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && nnz) e = cudaMemcpy(d_col, col, (size_t)nnz * 4, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && nnz) e = cudaMemcpy(d_val, val, (size_t)nnz * 16, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(d_rhs0, rhs0, (size_t)n * 16, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && n_l) e = cudaMemcpy(d_l, l_index, (size_t)n_l * 4, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemset(info, 0, 2 * sizeof(int));
  if (e != cudaSuccess) {
    cleanup();
    set_error(std::string("acpf_zbus_reduce: ") + cudaGetErrorString(e));
    return ACPF_ECUDA;
  }
  mark("upload");
  scatter_csr_colmajor<<<(n + 127) / 128, 128>>>(n, d_rp, d_col, (const double2*)d_val, a);
  fill_rhs<<<(unsigned)((nr + 255) / 256), 256>>>(n, n_l, d_l, d_rhs0, b);
  cusolverDnHandle_t h = nullptr;
  if (cusolverDnCreate(&h) != CUSOLVER_STATUS_SUCCESS) {
    cleanup();
    set_error("acpf_zbus_reduce: cusolverDnCreate failed");
    return ACPF_ECUDA;
  }
  mark("handle");
  int lwork = 0;
  cusolverStatus_t cs = cusolverDnZgetrf_bufferSize(h, n, n, (cuDoubleComplex*)a, n, &lwork);
  cuDoubleComplex* work = cs == CUSOLVER_STATUS_SUCCESS ? (cuDoubleComplex*)alloc((size_t)lwork * 16) : nullptr;
  if (cs == CUSOLVER_STATUS_SUCCESS && work)
    cs = cusolverDnZgetrf(h, n, n, (cuDoubleComplex*)a, n, work, ipiv, info);
  int h_info = 0;
  if (cs == CUSOLVER_STATUS_SUCCESS && work) cudaMemcpy(&h_info, info, sizeof(int), cudaMemcpyDeviceToHost);
  mark("getrf");
  int bad = 0;
  double min_piv = 0.0;
  if (cs == CUSOLVER_STATUS_SUCCESS && work) {
    diag_check<<<1, 256>>>(n, a, d_min, info + 1);
    cudaMemcpy(&min_piv, d_min, sizeof(double), cudaMemcpyDeviceToHost);
    cudaMemcpy(&bad, info + 1, sizeof(int), cudaMemcpyDeviceToHost);
    cudaMemset(info + 1, 0, sizeof(int));
    any_nonfinite<<<(unsigned)((nn + 255) / 256), 256>>>(nn, a, info + 1);
    int bad2 = 0;
    cudaMemcpy(&bad2, info + 1, sizeof(int), cudaMemcpyDeviceToHost);
    bad |= bad2;
  }
  if (min_pivot_out) *min_pivot_out = bad ? NAN : min_piv;
  if (cs != CUSOLVER_STATUS_SUCCESS || !work) {
    cusolverDnDestroy(h);
    cleanup();
    set_error("acpf_zbus_reduce: cuSOLVER getrf failed");
    return ACPF_ECUDA;
  }
  // the reference's test (distribution.py:458-473): non-finite factor or
  // min |U_ii| <= n eps max |Y_NN|
  double ymax = 0.0;
  for (int64_t k = 0; k < nnz; ++k) ymax = fmax(ymax, std::hypot(val[2 * k], val[2 * k + 1]));
  ymax = fmax(ymax, 2.2250738585072014e-308);
  if (bad || h_info > 0 || min_piv <= n * 2.220446049250313e-16 * ymax) {
    cusolverDnDestroy(h);
    cleanup();
    set_error("non-slack admittance block is numerically singular (isolated node-phase or zero-admittance island)");
    return ACPF_ESTRUCT;
  }
  mark("check");
  cusolverDnDestroy(h);
  if ((size_t)n * sizeof(double2) > 227 * 1024) {
    cleanup();
    set_error("acpf_zbus_reduce: network too large for the device triangular solves");
    return ACPF_ESTRUCT;
  }
  const int sm = n * (int)sizeof(double2);
  e = cudaFuncSetAttribute(lu_solve_columns, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  if (e == cudaSuccess) {
    lu_solve_columns<<<n_l + 1, 1024, sm>>>(n, a, ipiv, b);
    e = cudaGetLastError();
  }
  if (e != cudaSuccess) {
    cleanup();
    set_error(std::string("acpf_zbus_reduce: ") + cudaGetErrorString(e));
    return ACPF_ECUDA;
  }
  mark("getrs");
  // B is column-major n x (n_l + 1): Z[:, l_k] = B[:, k], v0 = B[:, n_l]
  std::vector<double2> hb(nr);
  e = cudaMemcpy(hb.data(), b, nr * sizeof(double2), cudaMemcpyDeviceToHost);
  cleanup();
  if (e != cudaSuccess) {
    set_error(std::string("acpf_zbus_reduce: ") + cudaGetErrorString(e));
    return ACPF_ECUDA;
  }
  for (int r = 0; r < n; ++r) {
    for (int k = 0; k < n_l; ++k) {
      zl_out[((size_t)r * n_l + k) * 2] = hb[(size_t)k * n + r].x;
      zl_out[((size_t)r * n_l + k) * 2 + 1] = hb[(size_t)k * n + r].y;
    }
    v0_out[2 * r] = hb[(size_t)n_l * n + r].x;
    v0_out[2 * r + 1] = hb[(size_t)n_l * n + r].y;
  }
  return ACPF_OK;
}

}  // namespace acpf
