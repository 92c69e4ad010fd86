// C-ABI entry points of libacpf.so (declared in include/acpf.h).
//
// Plans own device copies of the per-network model; solves stream the
// caller's batch through the fused kernels (nr_kernel.cu, zbus_kernel.cu),
// chunking when the batch would not fit the device workspace, staging host
// buffers through device memory when ACPF_HOST_PTRS is given.

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "acpf_internal.cuh"
#include "nr_symbolic.h"

namespace acpf {

static thread_local std::string g_error;

void set_error(const std::string& msg) { g_error = msg; }

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (dev != prev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

#define ACPF_CUDA(call)                                                              \
  do {                                                                               \
    cudaError_t e_ = (call);                                                         \
    if (e_ != cudaSuccess) {                                                         \
      set_error(std::string(#call) + ": " + cudaGetErrorString(e_));                 \
      return e_ == cudaErrorMemoryAllocation ? ACPF_ENOMEM : ACPF_ECUDA;             \
    }                                                                                \
  } while (0)

// Owning list of device allocations.
struct DevArena {
  std::vector<void*> ptrs;
  ~DevArena() { release(); }
  void release() {
    for (void* p : ptrs) cudaFree(p);
    ptrs.clear();
  }
  template <class T>
  cudaError_t upload(T** out, const T* host, size_t count) {
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, std::max<size_t>(1, count) * sizeof(T));
    if (e != cudaSuccess) return e;
    ptrs.push_back(p);
    if (count) e = cudaMemcpy(p, host, count * sizeof(T), cudaMemcpyHostToDevice);
    *out = static_cast<T*>(p);
    return e;
  }
  cudaError_t alloc(void** out, size_t bytes) {
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, std::max<size_t>(1, bytes));
    if (e != cudaSuccess) return e;
    ptrs.push_back(p);
    *out = p;
    return e;
  }
};

int64_t env_int(const char* name, int64_t dflt) {
  const char* v = std::getenv(name);
  if (!v || !*v) return dflt;
  return std::strtoll(v, nullptr, 10);
}

}  // namespace
}  // namespace acpf

using namespace acpf;

// Second concurrent chunk solver of the host-pointer path (lane 1; lane 0
// uses the plan's own workspace and graph cache): own stream, workspace,
// staging set, pinned active counter and graph cache.
struct NrLane {
  DevArena work, stage;
  NrWorkspace ws{};
  int64_t groups = 0;
  size_t stage_bytes = 0;
  void* stage_base = nullptr;
  int* host_active = nullptr;
  NrGraphCache graphs;
  cudaStream_t st = nullptr;
  cudaEvent_t ev_h2d = nullptr, ev_end = nullptr;
  // prefetch pipeline: inputs in / results out on their own copy streams,
  // two staging sets (the next chunk's H2D and the last chunk's D2H overlap
  // the current chunk's solve)
  cudaStream_t cs_in = nullptr, cs_out = nullptr;
  cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_done[2] = {nullptr, nullptr}, ev_out[2] = {nullptr, nullptr};
};

struct acpf_nr_plan {
  int device = 0;
  NrSymbolic sym;
  NrSchedule sch;
  NrHostSchedule hs{};
  NrDeviceModel dm{};
  DevArena model;
  DevArena work;
  NrWorkspace ws{};
  int64_t ws_groups = 0;
  int64_t bytes_per_group = 0;
  DevArena stage;
  size_t stage_bytes = 0;
  void* stage_base = nullptr;
  int* host_active = nullptr;
  NrGraphCache graphs;                  // captured Newton-step sequences
  std::vector<int32_t> h_tpos, h_qidx;  // host copies for scenario generation
  cudaStream_t copy_stream = nullptr;   // host-path H2D/D2H overlap
  cudaEvent_t ev_h2d[2] = {nullptr, nullptr}, ev_kend[2] = {nullptr, nullptr},
              ev_d2h[2] = {nullptr, nullptr};
  NrCertModel cert{};                   // acpf_nr_plan_set_branches (n_br < 0: not set)
  DevArena cert_arena;
  GmModel gm{};                         // acpf_nr_plan_set_fd (binv1 null: not set)
  DevArena gm_arena;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  double last_ms = 0.0;
  int last_launches = 0;
  NrLane lanes[2];                      // concurrent chunk solvers (host-pointer path)
  // device-pointer solves return without a host sync: their per-chunk events
  // and host-counted launches are resolved by acpf_nr_last_timing
  std::vector<cudaEvent_t> tev;
  int pending_chunks = 0, pending_launches = 0;
};

struct acpf_zbus_plan {
  int device = 0;
  int n_wye = 0, n_delta = 0;
  std::vector<int32_t> h_wye, h_dp, h_dq;  // reduced rows of the loads (certificates)
  double floor = 0.0;
  ZbCertModel cert{};                      // acpf_zbus_plan_set_network (rowptr null: not set)
  DevArena cert_arena;
  cudaStream_t copy_stream = nullptr;  // host-path H2D/D2H overlap
  cudaEvent_t ev_h2d[2] = {nullptr, nullptr}, ev_kend[2] = {nullptr, nullptr},
              ev_d2h[2] = {nullptr, nullptr};
  ZbDeviceModel dm{};
  DevArena model;
  DevArena stage;
  size_t stage_bytes = 0;
  void* stage_base = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  bool pending = false;  // last solve was a device-pointer (asynchronous) one
  double last_ms = 0.0;
  int last_launches = 0;
};

static void fill_info(const NrSymbolic& s, acpf_nr_plan_info* info, int64_t ws_bytes = -1) {
  info->n_bus = s.n_bus;
  info->n_theta = s.n_theta;
  info->n_q = s.n_q;
  info->n_j = s.n_j;
  info->nnz_y = (int32_t)s.nnz_y;
  info->nnz_j = (int32_t)s.nnz_j;
  info->nnz_lu = s.nnz_lu;
  info->n_pairs = s.n_pairs;
  info->group = kGroup;
  info->etree_height = s.etree_height;
  info->workspace_bytes_per_group =
      ws_bytes >= 0 ? ws_bytes
                    : (int64_t)kGroup * 8 * (s.nnz_lu + 3 * (int64_t)s.n_j + 9 * (int64_t)s.n_bus);
}

extern "C" {

const char* acpf_last_error(void) { return g_error.c_str(); }

int32_t acpf_abi_version(void) { return ACPF_ABI_VERSION; }

int32_t acpf_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

// ---------------------------------------------------------------------------
// Newton
// ---------------------------------------------------------------------------

acpf_status acpf_nr_plan_create(int32_t device, int32_t n_bus, const int32_t* y_rowptr,
                                const int32_t* y_col, const double* y_re, const double* y_im,
                                int32_t n_theta, const int32_t* theta_block, int32_t n_q,
                                const int32_t* q_block, const double* theta_init,
                                const double* vmag_init, const int32_t* perm,
                                acpf_nr_plan_t* out) {
  if (!out || n_bus <= 0 || !y_rowptr || !y_col || !y_re || !y_im || n_theta < 0 || n_q < 0 ||
      (n_theta && !theta_block) || (n_q && !q_block) || !theta_init || !vmag_init) {
    set_error("acpf_nr_plan_create: invalid argument");
    return ACPF_EINVAL;
  }
  *out = nullptr;
  acpf_nr_plan* p = new (std::nothrow) acpf_nr_plan();
  if (!p) {
    set_error("host allocation failed");
    return ACPF_ENOMEM;
  }
  try {
    // symbolic analysis on the bus graph: one 2x2 block unknown per non-slack
    // bus (theta_block order), Jacobian block pattern = Ybus pattern
    NrSymbolic first;
    build_nr_symbolic(first, n_bus, y_rowptr, y_col, n_theta, theta_block, 0, nullptr, perm);
    const std::vector<int32_t> lperm = level_sorted_perm(first);
    build_nr_symbolic(p->sym, n_bus, y_rowptr, y_col, n_theta, theta_block, 0, nullptr, lperm.data());
    build_nr_schedule(p->sym, y_rowptr, y_col, y_re, y_im, p->sch,
                      (int)env_int("ACPF_NR_TASK_ELEMS", 512),
                      env_int("ACPF_NR_COLUMN_STORE", 1) != 0,
                      (int)env_int("ACPF_NR_TAIL", kTailMaxRows));  // dense tail
    if (env_int("ACPF_DEBUG_SCHEDULE", 0)) {  // per-level shape of the factor schedule (stderr)
      const NrSchedule& sc = p->sch;
      for (int l = 0; l < sc.n_levels; ++l) {
        const int r0 = sc.level_ptr[l], r1 = sc.level_ptr[l + 1];
        std::fprintf(stderr, "level %d rows %d tasks %d maxl %d slots %d stream %d\n", l, r1 - r0,
                     sc.level_task_ptr[l + 1] - sc.level_task_ptr[l], sc.level_maxl[l],
                     sc.row_slot[r1] - sc.row_slot[r0], sc.row_sptr[r1] - sc.row_sptr[r0]);
      }
      std::fprintf(stderr, "tail rows %d (from row %d, level %d), %zu tail slots, back levels %d\n", sc.tail_T,
                   sc.tail_row0, sc.tail_level, sc.tail_slot.size() / 2, sc.n_blevels);
    }
  } catch (const std::exception& ex) {
    set_error(std::string("symbolic analysis: ") + ex.what());
    delete p;
    return ACPF_EINVAL;
  }
  p->device = device;
  DeviceGuard dg(device);
  const NrSymbolic& s = p->sym;
  const NrSchedule& sc = p->sch;
  const int64_t nnz = y_rowptr[n_bus];
  std::vector<double2> yv(nnz);
  for (int64_t e = 0; e < nnz; ++e) yv[e] = make_double2(y_re[e], y_im[e]);
  std::vector<int32_t> tpos(n_bus, -1), qidx(n_bus, -1);
  for (int k = 0; k < n_theta; ++k) tpos[theta_block[k]] = k;
  for (int k = 0; k < n_q; ++k) {
    if (q_block[k] < 0 || q_block[k] >= n_bus || tpos[q_block[k]] < 0) {
      set_error("acpf_nr_plan_create: q_block bus must be in theta_block");
      delete p;
      return ACPF_EINVAL;
    }
    qidx[q_block[k]] = k;
  }

  p->h_tpos = tpos;
  p->h_qidx = qidx;
  // LU of the flat-start Jacobian, shared by every scenario's first step
  std::vector<double> sh_vals, sh_s0;
  bool shared0 = false;
  if (env_int("ACPF_NR_SHARED0", 1)) {
    try {
      shared0 = nr_flat_start_factor(s, sc, n_bus, y_rowptr, y_col, y_re, y_im, qidx.data(), theta_init,
                                     vmag_init, sh_vals, &sh_s0);
    } catch (const std::exception&) {
      shared0 = false;
    }
  }
  std::vector<int32_t> sh_col(s.col.begin(), s.col.end()), sh_diag(s.diag.begin(), s.diag.end());
  NrDeviceModel& d = p->dm;
  d.n_bus = n_bus;
  d.n_theta = n_theta;
  d.n_q = n_q;
  d.n_rows = s.n_j;
  d.nnz_lu = s.nnz_lu;
  d.n_block = sc.n_block;
  d.n_scalar = sc.n_scalar;
  d.off_lu = sc.off_lu;
  d.off_yx = sc.off_yx;
  d.off_u = sc.off_u;
  d.off_e = sc.off_e;
  d.off_spec = sc.off_spec;
  d.off_th = sc.off_th;
  d.off_vm = sc.off_vm;
  p->cert.n_br = -1;
  p->hs.level_task_ptr = sc.level_task_ptr.data();
  p->hs.level_maxl = sc.level_maxl.data();
  p->hs.blevel_task_ptr = sc.blevel_task_ptr.data();
  p->hs.n_levels = sc.n_levels;
  p->hs.n_blevels = sc.n_blevels;
  p->hs.max_l = sc.max_l;
  p->hs.tail_level = sc.tail_level;
  p->hs.n_tail_class = (int)sc.tail_class_maxl.size();
  p->hs.tail_variant = (int)env_int("ACPF_NR_TAIL_VARIANT", 2);
  p->hs.tail_class_ptr = sc.tail_class_ptr.data();
  p->hs.tail_class_maxl = sc.tail_class_maxl.data();
  d.tail_row0 = sc.tail_row0;
  d.tail_T = sc.tail_T;
  d.n_tail_slot = (int)(sc.tail_slot.size() / 2);
  {
    // factor pipeline variant: the requested one if its shared memory (ring +
    // the longest L part of a row) fits one SM, else the next smaller one
    constexpr size_t kSmemMax = 227 * 1024;
    int v = (int)env_int("ACPF_NR_VARIANT", 3);
    v = v < 0 ? 0 : (v > 3 ? 3 : v);
    if (nr_smem_bytes(v, sc.max_l) > kSmemMax) v = 0;
    if (nr_smem_bytes(v, sc.max_l) > kSmemMax) {
      set_error("acpf_nr_plan_create: an L row of " + std::to_string(sc.max_l) +
                " blocks exceeds the shared-memory row buffer");
      delete p;
      return ACPF_ESTRUCT;
    }
    p->hs.variant = v;
  }
  cudaError_t e = cudaSuccess;
  auto up = [&](auto** dst, const auto* src, size_t cnt) {
    if (e == cudaSuccess) e = p->model.upload(dst, src, cnt);
  };
  up(const_cast<int32_t**>(&d.y_rowptr), y_rowptr, (size_t)n_bus + 1);
  up(const_cast<int32_t**>(&d.y_col), y_col, (size_t)nnz);
  up(const_cast<double2**>(&d.y_val), yv.data(), (size_t)nnz);
  up(const_cast<double**>(&d.theta_init), theta_init, (size_t)n_bus);
  up(const_cast<double**>(&d.vmag_init), vmag_init, (size_t)n_bus);
  up(const_cast<int32_t**>(&d.tpos), tpos.data(), (size_t)n_bus);
  up(const_cast<int32_t**>(&d.qidx), qidx.data(), (size_t)n_bus);
  up(const_cast<int32_t**>(&d.bus_row), sc.bus_row.data(), sc.bus_row.size());
  up(const_cast<int32_t**>(&d.asm_ptr), sc.asm_ptr.data(), sc.asm_ptr.size());
  up(const_cast<double2**>(&d.asm_y), reinterpret_cast<const double2*>(sc.asm_y.data()),
     sc.asm_y.size() / 2);
  up(const_cast<int32_t**>(&d.asm_j), sc.asm_j.data(), sc.asm_j.size());
  up(const_cast<int32_t**>(&d.asm_slot), sc.asm_slot.data(), sc.asm_slot.size());
  up(const_cast<uint32_t**>(&d.slot_info), sc.slot_info.data(), sc.slot_info.size());
  up(const_cast<int32_t**>(&d.slot_store), sc.slot_store.data(), sc.slot_store.size());
  up(const_cast<int32_t**>(&d.row_slot), sc.row_slot.data(), sc.row_slot.size());
  up(const_cast<int32_t**>(&d.row_sptr), sc.row_sptr.data(), sc.row_sptr.size());
  up(const_cast<int32_t**>(&d.task_row), sc.task_row.data(), sc.task_row.size());
  up(const_cast<int32_t**>(&d.btask_row), sc.btask_row.data(), sc.btask_row.size());
  up(const_cast<uint32_t**>(&d.brow), sc.brow.data(), sc.brow.size());
  up(const_cast<int32_t**>(&d.brow_sptr), sc.brow_sptr.data(), sc.brow_sptr.size());
  up(const_cast<uint32_t**>(&d.stream), sc.stream.data(), sc.stream.size());
  if (d.n_tail_slot)
    up(const_cast<int2**>(&d.tail_slot), reinterpret_cast<const int2*>(sc.tail_slot.data()),
       (size_t)d.n_tail_slot);
  if (!sc.tail_trow.empty()) up(const_cast<int32_t**>(&d.tail_trow), sc.tail_trow.data(), sc.tail_trow.size());
  if (shared0) {
    up(const_cast<double**>(&d.sh_vals), sh_vals.data(), sh_vals.size());
    up(const_cast<int32_t**>(&d.sh_col), sh_col.data(), sh_col.size());
    up(const_cast<int32_t**>(&d.sh_diag), sh_diag.data(), sh_diag.size());
    // the step-0 mismatch reads the flat-start S_i instead of gathering (the
    // V <= 0 exit check at step 0 then needs V > 0 everywhere at the flat start)
    bool vpos = true;
    for (int i = 0; i < n_bus; ++i) vpos = vpos && vmag_init[i] > 0.0;
    if (vpos && env_int("ACPF_NR_S0", 1))
      up(const_cast<double2**>(&d.sh_s0), reinterpret_cast<const double2*>(sh_s0.data()), (size_t)n_bus);
  }
  if (e == cudaSuccess) e = cudaEventCreate(&p->ev0);
  if (e == cudaSuccess) e = cudaEventCreate(&p->ev1);
  if (e != cudaSuccess) {
    set_error(std::string("acpf_nr_plan_create: ") + cudaGetErrorString(e));
    delete p;
    return e == cudaErrorMemoryAllocation ? ACPF_ENOMEM : ACPF_ECUDA;
  }
  p->bytes_per_group =
      (sc.n_block * 4 * kGroup + sc.n_scalar * kGroup) * 8 + (int64_t)nr_group_state_bytes();
  *out = p;
  return ACPF_OK;
}

acpf_status acpf_nr_ordering(int32_t n_bus, const int32_t* y_rowptr, const int32_t* y_col, int32_t n_theta,
                             const int32_t* theta_block, int32_t kind, int32_t* perm_out) {
  if (n_bus <= 0 || !y_rowptr || !y_col || n_theta <= 0 || !theta_block || !perm_out ||
      (kind != ACPF_ORDER_MIN_DEGREE && kind != ACPF_ORDER_MIN_FILL)) {
    set_error("acpf_nr_ordering: invalid argument");
    return ACPF_EINVAL;
  }
  try {
    NrSymbolic s;
    build_nr_symbolic(s, n_bus, y_rowptr, y_col, n_theta, theta_block, 0, nullptr, nullptr, kind);
    std::memcpy(perm_out, s.perm.data(), (size_t)n_theta * sizeof(int32_t));
  } catch (const std::exception& ex) {
    set_error(std::string("ordering: ") + ex.what());
    return ACPF_EINVAL;
  }
  return ACPF_OK;
}

acpf_status acpf_nr_analyze(int32_t n_bus, const int32_t* y_rowptr, const int32_t* y_col,
                            int32_t n_theta, const int32_t* theta_block, int32_t n_q,
                            const int32_t* q_block, const int32_t* perm, acpf_nr_plan_info* info) {
  if (n_bus <= 0 || !y_rowptr || !y_col || !info || (n_theta && !theta_block) || (n_q && !q_block)) {
    set_error("acpf_nr_analyze: invalid argument");
    return ACPF_EINVAL;
  }
  try {
    NrSymbolic s;
    (void)n_q;
    (void)q_block;
    build_nr_symbolic(s, n_bus, y_rowptr, y_col, n_theta, theta_block, 0, nullptr, perm);
    fill_info(s, info);
  } catch (const std::exception& ex) {
    set_error(std::string("symbolic analysis: ") + ex.what());
    return ACPF_EINVAL;
  }
  return ACPF_OK;
}

acpf_status acpf_nr_flat_start_solve(int32_t n_bus, const int32_t* y_rowptr, const int32_t* y_col,
                                     const double* y_re, const double* y_im, int32_t n_theta,
                                     const int32_t* theta_block, int32_t n_q, const int32_t* q_block,
                                     const double* theta_init, const double* vmag_init, const int32_t* perm,
                                     const double* rhs, double* x_out) {
  if (n_bus <= 0 || !y_rowptr || !y_col || !y_re || !y_im || n_theta < 0 || n_q < 0 ||
      (n_theta && !theta_block) || (n_q && !q_block) || !theta_init || !vmag_init || !rhs || !x_out) {
    set_error("acpf_nr_flat_start_solve: invalid argument");
    return ACPF_EINVAL;
  }
  try {
    // the same analysis, schedule and shared factor acpf_nr_plan_create builds
    NrSymbolic first, s;
    build_nr_symbolic(first, n_bus, y_rowptr, y_col, n_theta, theta_block, 0, nullptr, perm);
    const std::vector<int32_t> lperm = level_sorted_perm(first);
    build_nr_symbolic(s, n_bus, y_rowptr, y_col, n_theta, theta_block, 0, nullptr, lperm.data());
    NrSchedule sc;
    build_nr_schedule(s, y_rowptr, y_col, y_re, y_im, sc, 512, true);
    std::vector<int32_t> qidx(n_bus, -1);
    for (int k = 0; k < n_q; ++k) qidx[q_block[k]] = k;
    std::vector<double> v;
    if (!nr_flat_start_factor(s, sc, n_bus, y_rowptr, y_col, y_re, y_im, qidx.data(), theta_init, vmag_init, v)) {
      set_error("acpf_nr_flat_start_solve: zero pivot in the flat-start Jacobian");
      return ACPF_ESTRUCT;
    }
    // rhs / x in the reference's unknown order [theta_block; q_block]; a PV
    // bus's padded V unknown has the identity equation dV = 0
    const int nr = s.n_j;
    std::vector<double> y(2 * (size_t)nr, 0.0);
    for (int k = 0; k < n_theta; ++k) y[2 * (size_t)sc.bus_row[theta_block[k]]] = rhs[k];
    for (int k = 0; k < n_q; ++k) y[2 * (size_t)sc.bus_row[q_block[k]] + 1] = rhs[n_theta + k];
    for (int p = 0; p < nr; ++p) {  // y_p = inv(D_p) (b_p - sum_t L^_pt y_t)
      double a0 = y[2 * p], a1 = y[2 * p + 1];
      for (int64_t t = s.rowptr[p]; t < s.diag[p]; ++t) {
        const double* l = &v[4 * t];
        const double* yc = &y[2 * (size_t)s.col[t]];
        a0 -= l[0] * yc[0] + l[1] * yc[1];
        a1 -= l[2] * yc[0] + l[3] * yc[1];
      }
      const double* d = &v[4 * s.diag[p]];
      y[2 * p] = d[0] * a0 + d[1] * a1;
      y[2 * p + 1] = d[2] * a0 + d[3] * a1;
    }
    for (int p = nr - 1; p >= 0; --p) {  // x_p = y_p - sum_c U^_pc x_c
      for (int64_t t = s.diag[p] + 1; t < s.rowptr[p + 1]; ++t) {
        const double* u = &v[4 * t];
        const double* xc = &y[2 * (size_t)s.col[t]];
        y[2 * p] -= u[0] * xc[0] + u[1] * xc[1];
        y[2 * p + 1] -= u[2] * xc[0] + u[3] * xc[1];
      }
    }
    for (int k = 0; k < n_theta; ++k) x_out[k] = y[2 * (size_t)sc.bus_row[theta_block[k]]];
    for (int k = 0; k < n_q; ++k) x_out[n_theta + k] = y[2 * (size_t)sc.bus_row[q_block[k]] + 1];
  } catch (const std::exception& ex) {
    set_error(std::string("acpf_nr_flat_start_solve: ") + ex.what());
    return ACPF_EINVAL;
  }
  return ACPF_OK;
}

acpf_status acpf_nr_plan_info_get(acpf_nr_plan_t p, acpf_nr_plan_info* info) {
  if (!p || !info) {
    set_error("acpf_nr_plan_info_get: null argument");
    return ACPF_EINVAL;
  }
  fill_info(p->sym, info, p->bytes_per_group);
  return ACPF_OK;
}

acpf_status acpf_nr_plan_structure(acpf_nr_plan_t p, int32_t* perm_out, int64_t* lu_rowptr_out) {
  if (!p) {
    set_error("acpf_nr_plan_structure: null plan");
    return ACPF_EINVAL;
  }
  if (perm_out) std::memcpy(perm_out, p->sym.perm.data(), p->sym.perm.size() * sizeof(int32_t));
  if (lu_rowptr_out)
    std::memcpy(lu_rowptr_out, p->sym.rowptr.data(), p->sym.rowptr.size() * sizeof(int64_t));
  return ACPF_OK;
}

// the plan's graph cache unless ACPF_NR_GRAPHS=0 (direct launches)
static NrGraphCache* nr_graphs(acpf_nr_plan* p) {
  static const bool on = env_int("ACPF_NR_GRAPHS", 1) != 0;
  return on ? &p->graphs : nullptr;
}

static acpf_status nr_ensure_workspace(acpf_nr_plan* p, int64_t groups) {
  if (p->ws_groups >= groups) return ACPF_OK;
  p->work.release();
  p->ws_groups = 0;
  const size_t S = (size_t)groups * kGroup;
  NrWorkspace& w = p->ws;
  void* ptr = nullptr;
  bool ok = true;
  auto get = [&](size_t bytes) -> void* {
    if (!ok || p->work.alloc(&ptr, bytes) != cudaSuccess) {
      ok = false;
      return nullptr;
    }
    return ptr;
  };
  w.arena = (double*)get((size_t)groups * (p->sch.n_block * 4 + p->sch.n_scalar) * kGroup * 8);
  w.fmax_bits = (unsigned long long*)get(S * 8);
  w.flags = (int*)get(S * 4);
  w.status = (int*)get(S * 4);
  w.iters = (int*)get(S * 4);
  w.fout = (double*)get(S * 8);
  w.active = (uint8_t*)get(S);
  w.gactive = (int*)get((size_t)groups * 4);
  w.n_active = (int*)get(4);
  w.kstep = (int*)get(8);  // [0] Newton step, [1] kernels launched by the device loop
  if (ok) ok = cudaMemset(w.kstep, 0, 8) == cudaSuccess;
  if (!ok) {
    p->work.release();
    cudaGetLastError();
    set_error("acpf_nr_solve: device workspace allocation failed (" + std::to_string(groups) +
              " groups); lower ACPF_NR_CHUNK");
    return ACPF_ENOMEM;
  }
  if (!p->host_active) {
    if (cudaMallocHost(&p->host_active, sizeof(int)) != cudaSuccess) {
      cudaGetLastError();
      set_error("pinned host allocation failed");
      return ACPF_ENOMEM;
    }
  }
  w.host_active = p->host_active;
  w.groups = groups;
  p->ws_groups = groups;
  return ACPF_OK;
}

static acpf_status ensure_stage(DevArena& arena, size_t& have, void*& base, size_t bytes) {
  if (have >= bytes) return ACPF_OK;
  arena.release();
  have = 0;
  if (arena.alloc(&base, bytes) != cudaSuccess) {
    cudaGetLastError();
    set_error("staging allocation failed (" + std::to_string(bytes) + " bytes)");
    return ACPF_ENOMEM;
  }
  have = bytes;
  return ACPF_OK;
}

// Host-pointer solve pipelined over two staging sets: the H2D of chunk c+1
// and the D2H of chunk c-1 run on a copy stream while chunk c solves.
// kernels the device-side Newton loop launched since the last call (and reset)
static int nr_take_device_launches(const NrWorkspace& w) {
  int v[2] = {0, 0};
  if (!w.kstep || cudaMemcpy(v, w.kstep, sizeof v, cudaMemcpyDeviceToHost) != cudaSuccess) return 0;
  cudaMemset(w.kstep + 1, 0, sizeof(int));
  return v[1];
}

static acpf_status nr_solve_host(acpf_nr_plan* p, int64_t batch, int64_t chunk, const double* p_spec,
                                 const double* q_spec, double tol, int32_t max_newton, double* theta_out,
                                 double* vmag_out, uint8_t* converged, int32_t* iterations,
                                 double* final_mismatch_inf, int32_t* status, cudaStream_t st) {
  const NrDeviceModel& d = p->dm;
  if (!p->copy_stream) ACPF_CUDA(cudaStreamCreateWithFlags(&p->copy_stream, cudaStreamNonBlocking));
  for (int k = 0; k < 2; ++k) {
    if (!p->ev_h2d[k]) ACPF_CUDA(cudaEventCreateWithFlags(&p->ev_h2d[k], cudaEventDisableTiming));
    if (!p->ev_kend[k]) ACPF_CUDA(cudaEventCreateWithFlags(&p->ev_kend[k], cudaEventDisableTiming));
    if (!p->ev_d2h[k]) ACPF_CUDA(cudaEventCreateWithFlags(&p->ev_d2h[k], cudaEventDisableTiming));
  }
  cudaStream_t cs = p->copy_stream;
  const size_t set_b = (size_t)chunk * ((size_t)(d.n_theta + d.n_q) * 8 + (size_t)d.n_bus * 16 + 8 + 4 + 4 + 1) + 256;
  acpf_status rc = ensure_stage(p->stage, p->stage_bytes, p->stage_base, 2 * set_b);
  if (rc != ACPF_OK) return rc;
  struct Set {
    double *ps, *qs, *th, *vm, *fn;
    int32_t *it, *stt;
    uint8_t* cv;
  } sets[2];
  for (int k = 0; k < 2; ++k) {
    char* b = (char*)p->stage_base + k * set_b;
    auto take = [&](size_t bytes) {
      char* r = b;
      b += (bytes + 15) & ~(size_t)15;
      return r;
    };
    sets[k].ps = (double*)take((size_t)chunk * d.n_theta * 8);
    sets[k].qs = (double*)take((size_t)chunk * d.n_q * 8);
    sets[k].th = (double*)take((size_t)chunk * d.n_bus * 8);
    sets[k].vm = (double*)take((size_t)chunk * d.n_bus * 8);
    sets[k].fn = (double*)take((size_t)chunk * 8);
    sets[k].it = (int32_t*)take((size_t)chunk * 4);
    sets[k].stt = (int32_t*)take((size_t)chunk * 4);
    sets[k].cv = (uint8_t*)take((size_t)chunk);
  }
  const int64_t n_chunks = (batch + chunk - 1) / chunk;
  auto h2d = [&](int64_t c) -> acpf_status {
    const Set& S = sets[c & 1];
    const int64_t s0 = c * chunk, nb = std::min(chunk, batch - s0);
    if (d.n_theta)
      ACPF_CUDA(cudaMemcpyAsync(S.ps, p_spec + s0 * d.n_theta, nb * d.n_theta * 8, cudaMemcpyHostToDevice, cs));
    if (d.n_q) ACPF_CUDA(cudaMemcpyAsync(S.qs, q_spec + s0 * d.n_q, nb * d.n_q * 8, cudaMemcpyHostToDevice, cs));
    ACPF_CUDA(cudaEventRecord(p->ev_h2d[c & 1], cs));
    return ACPF_OK;
  };
  ACPF_CUDA(cudaStreamWaitEvent(cs, p->ev1, 0));  // a previous call's work on st is done with the sets
  if ((rc = h2d(0)) != ACPF_OK) return rc;
  float total_ms = 0.0f;
  int launches = 0;
  for (int64_t c = 0; c < n_chunks; ++c) {
    const Set& S = sets[c & 1];
    const int64_t s0 = c * chunk, nb = std::min(chunk, batch - s0);
    ACPF_CUDA(cudaStreamWaitEvent(st, p->ev_h2d[c & 1], 0));
    if (c >= 2) ACPF_CUDA(cudaStreamWaitEvent(st, p->ev_d2h[c & 1], 0));  // outputs of chunk c-2 read
    if (c + 1 < n_chunks && (rc = h2d(c + 1)) != ACPF_OK) return rc;  // queued behind D2H(c-1) on cs
    NrBatchIO io{};
    io.batch = nb;
    io.p_spec = S.ps;
    io.q_spec = S.qs;
    io.theta_out = S.th;
    io.vmag_out = S.vm;
    io.fnorm = S.fn;
    io.iterations = S.it;
    io.status = S.stt;
    io.converged = S.cv;
    ACPF_CUDA(cudaEventRecord(p->ev0, st));
    int nl = 0;
    NrWorkspace wsb = p->ws;
    wsb.groups = (nb + kGroup - 1) / kGroup;
    ACPF_CUDA(launch_nr_newton(d, p->hs, wsb, io, tol, max_newton, st, &nl, nr_graphs(p)));
    ACPF_CUDA(cudaEventRecord(p->ev1, st));
    ACPF_CUDA(cudaEventRecord(p->ev_kend[c & 1], st));
    launches += nl;
    ACPF_CUDA(cudaStreamWaitEvent(cs, p->ev_kend[c & 1], 0));
    ACPF_CUDA(cudaMemcpyAsync(theta_out + s0 * d.n_bus, S.th, nb * d.n_bus * 8, cudaMemcpyDeviceToHost, cs));
    ACPF_CUDA(cudaMemcpyAsync(vmag_out + s0 * d.n_bus, S.vm, nb * d.n_bus * 8, cudaMemcpyDeviceToHost, cs));
    if (final_mismatch_inf)
      ACPF_CUDA(cudaMemcpyAsync(final_mismatch_inf + s0, S.fn, nb * 8, cudaMemcpyDeviceToHost, cs));
    if (iterations) ACPF_CUDA(cudaMemcpyAsync(iterations + s0, S.it, nb * 4, cudaMemcpyDeviceToHost, cs));
    if (status) ACPF_CUDA(cudaMemcpyAsync(status + s0, S.stt, nb * 4, cudaMemcpyDeviceToHost, cs));
    if (converged) ACPF_CUDA(cudaMemcpyAsync(converged + s0, S.cv, nb, cudaMemcpyDeviceToHost, cs));
    ACPF_CUDA(cudaEventRecord(p->ev_d2h[c & 1], cs));
    ACPF_CUDA(cudaEventSynchronize(p->ev1));
    float ms = 0.0f;
    ACPF_CUDA(cudaEventElapsedTime(&ms, p->ev0, p->ev1));
    total_ms += ms;
  }
  ACPF_CUDA(cudaStreamSynchronize(cs));
  ACPF_CUDA(cudaStreamSynchronize(st));
  p->last_ms = total_ms;
  p->last_launches = launches + nr_take_device_launches(p->ws);
  return ACPF_OK;
}

static acpf_status nr_lane_workspace(acpf_nr_plan* p, NrLane& L, int64_t groups) {
  if (L.groups >= groups) return ACPF_OK;
  L.work.release();
  L.groups = 0;
  const size_t S = (size_t)groups * kGroup;
  NrWorkspace& w = L.ws;
  void* ptr = nullptr;
  bool ok = true;
  auto get = [&](size_t bytes) -> void* {
    if (!ok || L.work.alloc(&ptr, bytes) != cudaSuccess) {
      ok = false;
      return nullptr;
    }
    return ptr;
  };
  w.arena = (double*)get((size_t)groups * (p->sch.n_block * 4 + p->sch.n_scalar) * kGroup * 8);
  w.fmax_bits = (unsigned long long*)get(S * 8);
  w.flags = (int*)get(S * 4);
  w.status = (int*)get(S * 4);
  w.iters = (int*)get(S * 4);
  w.fout = (double*)get(S * 8);
  w.active = (uint8_t*)get(S);
  w.gactive = (int*)get((size_t)groups * 4);
  w.n_active = (int*)get(4);
  w.kstep = (int*)get(8);  // [0] Newton step, [1] kernels launched by the device loop
  if (ok) ok = cudaMemset(w.kstep, 0, 8) == cudaSuccess;
  if (!ok) {
    L.work.release();
    cudaGetLastError();
    set_error("acpf_nr_solve: device workspace allocation failed (" + std::to_string(groups) +
              " groups, second chunk lane); lower ACPF_NR_CHUNK");
    return ACPF_ENOMEM;
  }
  L.groups = groups;
  return ACPF_OK;
}

// Host-pointer solve on two concurrent chunk lanes: even chunks on lane 0,
// odd chunks on lane 1, each lane a stream that copies its chunk in, solves it
// (its own host thread drives the Newton loop, which waits for the active
// count every step) and copies the results out. Lane 1's first H2D is queued
// behind lane 0's, so lane 0 starts solving while lane 1's inputs arrive and
// lane 0's D2H runs while lane 1 finishes; the two solves share the GPU, so
// their level launches fill each other's tails (a chunk solved alone loses
// ~10% in launch tails against the whole batch).
constexpr acpf_status kLaneFallback = 1;  // internal: second lane unavailable

static acpf_status nr_solve_lanes(acpf_nr_plan* p, int64_t batch, int64_t chunk, const double* p_spec,
                                  const double* q_spec, double tol, int32_t max_newton, double* theta_out,
                                  double* vmag_out, uint8_t* converged, int32_t* iterations,
                                  double* final_mismatch_inf, int32_t* status, cudaStream_t st) {
  const NrDeviceModel& d = p->dm;
  const int64_t groups = chunk / kGroup;
  // chunk boundaries: a short first and last chunk (the first H2D and the
  // last D2H are the only copies nothing overlaps), full chunks between; the
  // two lanes take alternate chunks and end up with equal shares
  std::vector<int64_t> cbeg;
  {
    // ACPF_NR_EDGE_DIV: edge chunk = B / div (10: 314-315 ms on the device timeline at 65,536 vs 322-325 for 8)
    static const int64_t edge_div = std::max<int64_t>(2, env_int("ACPF_NR_EDGE_DIV", 10));
    const int64_t edge = ((std::min(chunk, batch / edge_div) + kGroup - 1) / kGroup) * kGroup;
    if (batch > 2 * chunk || edge < 1024 || env_int("ACPF_NR_EDGE_CHUNKS", 1) == 0) {
      for (int64_t s0 = 0; s0 < batch; s0 += chunk) cbeg.push_back(s0);
    } else {  // [edge, (B - 2 edge) / 2, (B - 2 edge) / 2, edge]
      const int64_t mid = ((batch - 2 * edge) / 2 + kGroup - 1) / kGroup * kGroup;
      for (int64_t s0 : {(int64_t)0, edge, edge + mid, batch - edge}) cbeg.push_back(s0);
    }
    cbeg.push_back(batch);
  }
  const int64_t n_chunks = (int64_t)cbeg.size() - 1;
  const size_t set_b = (size_t)chunk * ((size_t)(d.n_theta + d.n_q) * 8 + (size_t)d.n_bus * 16 + 8 + 4 + 4 + 1) + 256;
  struct Set {
    double *ps, *qs, *th, *vm, *fn;
    int32_t *it, *stt;
    uint8_t* cv;
  } sets[2][2];  // [lane][staging set]
  NrWorkspace ws[2];
  NrGraphCache* graphs[2] = {nullptr, nullptr};
  const int n_lanes = n_chunks > 1 ? 2 : 1;  // one chunk: no second workspace
  for (int k = 0; k < n_lanes; ++k) {
    NrLane& L = p->lanes[k];
    if (!L.st) ACPF_CUDA(cudaStreamCreateWithFlags(&L.st, cudaStreamNonBlocking));
    if (!L.cs_in) ACPF_CUDA(cudaStreamCreateWithFlags(&L.cs_in, cudaStreamNonBlocking));
    if (!L.cs_out) ACPF_CUDA(cudaStreamCreateWithFlags(&L.cs_out, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      if (!L.ev_in[i]) ACPF_CUDA(cudaEventCreateWithFlags(&L.ev_in[i], cudaEventDisableTiming));
      if (!L.ev_done[i]) ACPF_CUDA(cudaEventCreateWithFlags(&L.ev_done[i], cudaEventDisableTiming));
      if (!L.ev_out[i]) ACPF_CUDA(cudaEventCreateWithFlags(&L.ev_out[i], cudaEventDisableTiming));
    }
    if (!L.ev_h2d) ACPF_CUDA(cudaEventCreateWithFlags(&L.ev_h2d, cudaEventDisableTiming));
    if (!L.ev_end) ACPF_CUDA(cudaEventCreate(&L.ev_end));
    // two staging sets when the lane solves more than one chunk
    const int nset = n_chunks > 2 ? 2 : 1;
    acpf_status rc = ensure_stage(L.stage, L.stage_bytes, L.stage_base, nset * set_b);
    if (rc != ACPF_OK) return rc;
    if (k == 0) {  // lane 0: the plan's workspace (sized for the chunk by the caller) and graphs
      ws[0] = p->ws;
      graphs[0] = nr_graphs(p);
    } else {
      // lane 1's workspace; if it does not fit, the caller falls back to the
      // single-workspace copy-stream pipeline (nr_solve_host)
      if ((rc = nr_lane_workspace(p, L, groups)) != ACPF_OK) return kLaneFallback;
      if (!L.host_active && cudaMallocHost(&L.host_active, sizeof(int)) != cudaSuccess) {
        cudaGetLastError();
        set_error("pinned host allocation failed");
        return ACPF_ENOMEM;
      }
      ws[1] = L.ws;
      ws[1].host_active = L.host_active;
      graphs[1] = nr_graphs(p) ? &L.graphs : nullptr;
    }
    for (int i = 0; i < 2; ++i) {
      char* b = (char*)L.stage_base + (size_t)(i % nset) * set_b;
      auto take = [&](size_t bytes) {
        char* r = b;
        b += (bytes + 15) & ~(size_t)15;
        return r;
      };
      Set& S = sets[k][i];
      S.ps = (double*)take((size_t)chunk * d.n_theta * 8);
      S.qs = (double*)take((size_t)chunk * d.n_q * 8);
      S.th = (double*)take((size_t)chunk * d.n_bus * 8);
      S.vm = (double*)take((size_t)chunk * d.n_bus * 8);
      S.fn = (double*)take((size_t)chunk * 8);
      S.it = (int32_t*)take((size_t)chunk * 4);
      S.stt = (int32_t*)take((size_t)chunk * 4);
      S.cv = (uint8_t*)take((size_t)chunk);
    }
  }
  // chunk c runs on lane c & 1 as that lane's (c >> 1)-th chunk, staging set (c >> 1) & 1
  auto set_of = [&](int64_t c) -> Set& { return sets[c & 1][(c >> 1) & 1]; };
  auto h2d = [&](int64_t c, cudaStream_t s) -> acpf_status {
    const Set& S = set_of(c);
    const int64_t s0 = cbeg[c], nb = cbeg[c + 1] - cbeg[c];
    if (d.n_theta)
      ACPF_CUDA(cudaMemcpyAsync(S.ps, p_spec + s0 * d.n_theta, nb * d.n_theta * 8, cudaMemcpyHostToDevice, s));
    if (d.n_q) ACPF_CUDA(cudaMemcpyAsync(S.qs, q_spec + s0 * d.n_q, nb * d.n_q * 8, cudaMemcpyHostToDevice, s));
    return ACPF_OK;
  };
  auto d2h = [&](int64_t c, cudaStream_t s) -> acpf_status {
    const Set& S = set_of(c);
    const int64_t c0 = cbeg[c], nb = cbeg[c + 1] - cbeg[c];
    ACPF_CUDA(cudaMemcpyAsync(theta_out + c0 * d.n_bus, S.th, nb * d.n_bus * 8, cudaMemcpyDeviceToHost, s));
    ACPF_CUDA(cudaMemcpyAsync(vmag_out + c0 * d.n_bus, S.vm, nb * d.n_bus * 8, cudaMemcpyDeviceToHost, s));
    if (final_mismatch_inf) ACPF_CUDA(cudaMemcpyAsync(final_mismatch_inf + c0, S.fn, nb * 8, cudaMemcpyDeviceToHost, s));
    if (iterations) ACPF_CUDA(cudaMemcpyAsync(iterations + c0, S.it, nb * 4, cudaMemcpyDeviceToHost, s));
    if (status) ACPF_CUDA(cudaMemcpyAsync(status + c0, S.stt, nb * 4, cudaMemcpyDeviceToHost, s));
    if (converged) ACPF_CUDA(cudaMemcpyAsync(converged + c0, S.cv, nb, cudaMemcpyDeviceToHost, s));
    return ACPF_OK;
  };
  // order after the caller's stream; lane 0's first H2D goes before lane 1's
  ACPF_CUDA(cudaEventRecord(p->ev0, st));
  for (int k = 0; k < n_lanes; ++k) {
    NrLane& L = p->lanes[k];
    ACPF_CUDA(cudaStreamWaitEvent(L.st, p->ev0, 0));
    ACPF_CUDA(cudaStreamWaitEvent(L.cs_in, p->ev0, 0));
    ACPF_CUDA(cudaStreamWaitEvent(L.cs_out, p->ev0, 0));
  }
  {
    acpf_status rc = h2d(0, p->lanes[0].cs_in);
    if (rc != ACPF_OK) return rc;
    ACPF_CUDA(cudaEventRecord(p->lanes[0].ev_in[0], p->lanes[0].cs_in));
    if (n_lanes > 1) {
      ACPF_CUDA(cudaStreamWaitEvent(p->lanes[1].cs_in, p->lanes[0].ev_in[0], 0));
      if ((rc = h2d(1, p->lanes[1].cs_in)) != ACPF_OK) return rc;
      ACPF_CUDA(cudaEventRecord(p->lanes[1].ev_in[0], p->lanes[1].cs_in));
    }
  }
  acpf_status lrc[2] = {ACPF_OK, ACPF_OK};
  std::string lerr[2];
  int lnl[2] = {0, 0};
  // ACPF_NR_TRACE=1: per-chunk event timeline of the lanes on stderr
  static const bool trace = env_int("ACPF_NR_TRACE", 0) != 0;
  std::vector<cudaEvent_t> tev(trace ? 4 * n_chunks : 0);
  for (auto& e : tev) ACPF_CUDA(cudaEventCreate(&e));
  auto mark = [&](int64_t c, int what, cudaStream_t s) {
    if (trace) cudaEventRecord(tev[4 * c + what], s);
  };
  auto run = [&](int k) {
    cudaSetDevice(p->device);
    NrLane& L = p->lanes[k];
    auto body = [&]() -> acpf_status {
      for (int64_t c = k; c < n_chunks; c += 2) {
        const int j = (int)((c >> 1) & 1);
        const Set& S = set_of(c);
        const int64_t nb = cbeg[c + 1] - cbeg[c];
        // the solve waits for its inputs only
        ACPF_CUDA(cudaStreamWaitEvent(L.st, L.ev_in[j], 0));
        mark(c, 1, L.st);
        NrBatchIO io{};
        io.batch = nb;
        io.p_spec = S.ps;
        io.q_spec = S.qs;
        io.theta_out = S.th;
        io.vmag_out = S.vm;
        io.fnorm = S.fn;
        io.iterations = S.it;
        io.status = S.stt;
        io.converged = S.cv;
        NrWorkspace wsb = ws[k];
        wsb.groups = (nb + kGroup - 1) / kGroup;
        int nl = 0;
        ACPF_CUDA(launch_nr_newton(d, p->hs, wsb, io, tol, max_newton, L.st, &nl, graphs[k]));
        lnl[k] += nl;
        mark(c, 2, L.st);
        ACPF_CUDA(cudaEventRecord(L.ev_done[j], L.st));
        // prefetch the lane's next chunk into the other staging set once
        // that set's previous results have been copied out
        if (c + 2 < n_chunks) {
          const int jn = j ^ 1;
          if (c >= 2) ACPF_CUDA(cudaStreamWaitEvent(L.cs_in, L.ev_out[jn], 0));
          mark(c + 2, 0, L.cs_in);
          acpf_status r = h2d(c + 2, L.cs_in);
          if (r != ACPF_OK) return r;
          ACPF_CUDA(cudaEventRecord(L.ev_in[jn], L.cs_in));
        }
        // results out on the output copy stream
        ACPF_CUDA(cudaStreamWaitEvent(L.cs_out, L.ev_done[j], 0));
        acpf_status r = d2h(c, L.cs_out);
        if (r != ACPF_OK) return r;
        ACPF_CUDA(cudaEventRecord(L.ev_out[j], L.cs_out));
        mark(c, 3, L.cs_out);
      }
      ACPF_CUDA(cudaStreamWaitEvent(L.st, L.ev_out[0], 0));
      ACPF_CUDA(cudaStreamWaitEvent(L.st, L.ev_out[1], 0));
      ACPF_CUDA(cudaEventRecord(L.ev_end, L.st));
      ACPF_CUDA(cudaStreamSynchronize(L.st));
      return ACPF_OK;
    };
    lrc[k] = body();
    if (lrc[k] != ACPF_OK) lerr[k] = acpf_last_error();
  };
  if (n_chunks > 1) {
    std::thread t1(run, 1);
    run(0);
    t1.join();
  } else {
    run(0);
  }
  for (int k = 0; k < n_lanes; ++k)
    if (lrc[k] != ACPF_OK) {
      set_error(lerr[k]);
      return lrc[k];
    }
  if (trace) {
    for (int64_t c = 0; c < n_chunks; ++c) {
      float t[4] = {-1, -1, -1, -1};
      for (int i = c >= 2 ? 0 : 1; i < 4; ++i) cudaEventElapsedTime(&t[i], p->ev0, tev[4 * c + i]);
      std::fprintf(stderr, "lane %d chunk %lld (%lld scenarios): h2d@%.1f solve %.1f-%.1f d2h-end %.1f ms\n",
                   (int)(c & 1), (long long)c, (long long)(cbeg[c + 1] - cbeg[c]), t[0], t[1], t[2], t[3]);
    }
    for (auto& e : tev) cudaEventDestroy(e);
  }
  float ms = 0.0f, ms1 = 0.0f;
  ACPF_CUDA(cudaEventElapsedTime(&ms, p->ev0, p->lanes[0].ev_end));
  if (n_chunks > 1) ACPF_CUDA(cudaEventElapsedTime(&ms1, p->ev0, p->lanes[1].ev_end));
  p->last_ms = std::max(ms, ms1);  // wall time of the whole host-pointer solve incl. copies (acpf.h)
  p->last_launches = lnl[0] + lnl[1] + nr_take_device_launches(ws[0]) +
                     (n_lanes > 1 ? nr_take_device_launches(ws[1]) : 0);
  return ACPF_OK;
}

static acpf_status nr_solve_impl(acpf_nr_plan_t p, int64_t batch, const double* p_spec, const double* q_spec,
                                 const double* theta_start, const double* vmag_start, double tol_mismatch,
                                 int32_t max_newton, double* theta_out, double* vmag_out, uint8_t* converged,
                                 int32_t* iterations, double* final_mismatch_inf, int32_t* status,
                                 uint32_t flags, void* cuda_stream);

acpf_status acpf_nr_solve(acpf_nr_plan_t p, int64_t batch, const double* p_spec,
                          const double* q_spec, double tol_mismatch, int32_t max_newton,
                          double* theta_out, double* vmag_out, uint8_t* converged,
                          int32_t* iterations, double* final_mismatch_inf, int32_t* status,
                          uint32_t flags, void* cuda_stream) {
  return nr_solve_impl(p, batch, p_spec, q_spec, nullptr, nullptr, tol_mismatch, max_newton, theta_out, vmag_out,
                       converged, iterations, final_mismatch_inf, status, flags, cuda_stream);
}

acpf_status acpf_nr_solve_start(acpf_nr_plan_t p, int64_t batch, const double* p_spec, const double* q_spec,
                                const double* theta_start, const double* vmag_start, double tol_mismatch,
                                int32_t max_newton, double* theta_out, double* vmag_out, uint8_t* converged,
                                int32_t* iterations, double* final_mismatch_inf, int32_t* status,
                                uint32_t flags, void* cuda_stream) {
  if (!theta_start || !vmag_start) {
    set_error("acpf_nr_solve_start: theta_start and vmag_start are required");
    return ACPF_EINVAL;
  }
  return nr_solve_impl(p, batch, p_spec, q_spec, theta_start, vmag_start, tol_mismatch, max_newton, theta_out,
                       vmag_out, converged, iterations, final_mismatch_inf, status, flags, cuda_stream);
}

static acpf_status nr_solve_impl(acpf_nr_plan_t p, int64_t batch, const double* p_spec, const double* q_spec,
                                 const double* theta_start, const double* vmag_start, double tol_mismatch,
                                 int32_t max_newton, double* theta_out, double* vmag_out, uint8_t* converged,
                                 int32_t* iterations, double* final_mismatch_inf, int32_t* status,
                                 uint32_t flags, void* cuda_stream) {
  if (!p || batch < 0 || !theta_out || !vmag_out || max_newton < 1 || !(tol_mismatch > 0) ||
      (p->dm.n_theta && !p_spec) || (p->dm.n_q && !q_spec) || flags > 1u) {
    set_error("acpf_nr_solve: invalid argument");
    return ACPF_EINVAL;
  }
  const bool warm = theta_start != nullptr;
  if (batch == 0) return ACPF_OK;
  DeviceGuard dg(p->device);
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const NrDeviceModel& d = p->dm;
  const bool dev_ptrs = flags & ACPF_DEVICE_PTRS;

  int64_t chunk = env_int("ACPF_NR_CHUNK", 0);
  const int pipeline = (int)env_int("ACPF_NR_PIPELINE", 2);  // 0 serial, 1 copy stream, 2 two lanes
  // host buffers with >= 2 chunks on two lanes hold two workspaces at once
  const bool two_lanes = !dev_ptrs && pipeline == 2 && batch >= 2 * 8192;
  if (chunk <= 0) {
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    // the plan's existing workspaces are reusable, so they count as free
    const int64_t have_groups = p->ws_groups + (two_lanes ? p->lanes[1].groups : 0);
    int64_t budget = (int64_t)(free_b * 0.6) + have_groups * p->bytes_per_group;
    if (two_lanes) budget /= 2;
    int64_t groups = std::max<int64_t>(1, budget / std::max<int64_t>(1, p->bytes_per_group));
    groups = std::min<int64_t>(groups, env_int("ACPF_NR_CHUNK_GROUPS", 16384));
    chunk = groups * kGroup;
    // equal chunks: no short last chunk running its levels on a partial wave
    // (2^20 device-resident: 14 chunks of ~75k, 233k/s -> 240k/s)
    const int64_t n_chunks = (batch + chunk - 1) / chunk;
    chunk = std::min<int64_t>(chunk, (batch + n_chunks - 1) / n_chunks);
  }
  chunk = std::min<int64_t>(chunk, batch);
  // host buffers: at least two chunks so transfers overlap the solves
  if (!dev_ptrs && env_int("ACPF_NR_CHUNK", 0) <= 0 && batch >= 2 * 8192) {
    chunk = std::min<int64_t>(chunk, (batch + 1) / 2);
    if (pipeline == 2) chunk = std::min<int64_t>(chunk, 32768);  // two lane workspaces in flight
  }
  chunk = ((chunk + kGroup - 1) / kGroup) * kGroup;
  const int64_t groups = chunk / kGroup;
  acpf_status rc = nr_ensure_workspace(p, groups);
  if (rc != ACPF_OK) return rc;

  if (!dev_ptrs && pipeline == 2 && !warm) {
    rc = nr_solve_lanes(p, batch, chunk, p_spec, q_spec, tol_mismatch, max_newton, theta_out, vmag_out,
                        converged, iterations, final_mismatch_inf, status, st);
    if (rc != kLaneFallback) return rc;
    cudaGetLastError();  // lane 1 did not fit: one workspace, copy-stream pipeline
    return nr_solve_host(p, batch, chunk, p_spec, q_spec, tol_mismatch, max_newton, theta_out, vmag_out,
                         converged, iterations, final_mismatch_inf, status, st);
  }
  if (!dev_ptrs && pipeline == 1 && !warm)
    return nr_solve_host(p, batch, chunk, p_spec, q_spec, tol_mismatch, max_newton, theta_out, vmag_out,
                         converged, iterations, final_mismatch_inf, status, st);
  // per-scenario byte sizes
  const size_t in_b = (size_t)(d.n_theta + d.n_q) * 8 + (warm ? (size_t)d.n_bus * 16 : 0);
  const size_t out_b = (size_t)d.n_bus * 16 + 1 + 4 + 8 + 4;
  if (!dev_ptrs) {
    rc = ensure_stage(p->stage, p->stage_bytes, p->stage_base, (size_t)chunk * (in_b + out_b) + 512);
    if (rc != ACPF_OK) return rc;
  }
  float total_ms = 0.0f;
  int launches = 0;
  int64_t ci = 0;  // chunk index
  if (dev_ptrs) {
    // asynchronous w.r.t. the host (like any stream-ordered CUDA library
    // call): the device launch counter restarts for this solve
    ACPF_CUDA(cudaMemsetAsync(p->ws.kstep + 1, 0, sizeof(int), st));
    p->pending_chunks = 0;
  }
  for (int64_t s0 = 0; s0 < batch; s0 += chunk, ++ci) {
    const int64_t nb = std::min(chunk, batch - s0);
    NrBatchIO io{};
    io.batch = nb;
    while (p->tev.size() < (size_t)(2 * ci + 2)) {
      cudaEvent_t e;
      ACPF_CUDA(cudaEventCreate(&e));
      p->tev.push_back(e);
    }
    if (dev_ptrs) {
      io.p_spec = p_spec ? p_spec + s0 * d.n_theta : nullptr;
      io.q_spec = q_spec ? q_spec + s0 * d.n_q : nullptr;
      if (warm) {
        io.theta_start = theta_start + s0 * d.n_bus;
        io.vmag_start = vmag_start + s0 * d.n_bus;
      }
      io.theta_out = theta_out + s0 * d.n_bus;
      io.vmag_out = vmag_out + s0 * d.n_bus;
      io.converged = converged ? converged + s0 : nullptr;
      io.iterations = iterations ? iterations + s0 : nullptr;
      io.fnorm = final_mismatch_inf ? final_mismatch_inf + s0 : nullptr;
      io.status = status ? status + s0 : nullptr;
    } else {
      char* b = (char*)p->stage_base;
      double* ps = (double*)b;
      b += (size_t)chunk * d.n_theta * 8;
      double* qs = (double*)b;
      b += (size_t)chunk * d.n_q * 8;
      double* th = (double*)b;
      b += (size_t)chunk * d.n_bus * 8;
      double* vm = (double*)b;
      b += (size_t)chunk * d.n_bus * 8;
      double* fn = (double*)b;
      b += (size_t)chunk * 8;
      int32_t* it = (int32_t*)b;
      b += (size_t)chunk * 4;
      int32_t* stt = (int32_t*)b;
      b += (size_t)chunk * 4;
      uint8_t* cv = (uint8_t*)b;
      b += (size_t)chunk;
      if (warm) {  // start state staged after the outputs (16-byte aligned)
        b = (char*)(((uintptr_t)b + 15) & ~(uintptr_t)15);
        double* ths = (double*)b;
        b += (size_t)chunk * d.n_bus * 8;
        double* vms = (double*)b;
        ACPF_CUDA(cudaMemcpyAsync(ths, theta_start + s0 * d.n_bus, nb * d.n_bus * 8, cudaMemcpyHostToDevice, st));
        ACPF_CUDA(cudaMemcpyAsync(vms, vmag_start + s0 * d.n_bus, nb * d.n_bus * 8, cudaMemcpyHostToDevice, st));
        io.theta_start = ths;
        io.vmag_start = vms;
      }
      if (d.n_theta)
        ACPF_CUDA(cudaMemcpyAsync(ps, p_spec + s0 * d.n_theta, nb * d.n_theta * 8, cudaMemcpyHostToDevice, st));
      if (d.n_q)
        ACPF_CUDA(cudaMemcpyAsync(qs, q_spec + s0 * d.n_q, nb * d.n_q * 8, cudaMemcpyHostToDevice, st));
      io.p_spec = ps;
      io.q_spec = qs;
      io.theta_out = th;
      io.vmag_out = vm;
      io.fnorm = fn;
      io.iterations = it;
      io.status = stt;
      io.converged = cv;
    }
    ACPF_CUDA(cudaEventRecord(p->tev[2 * ci], st));
    int nl = 0;
    NrWorkspace wsb = p->ws;  // capacity may exceed this chunk: index by the chunk's groups
    wsb.groups = (nb + kGroup - 1) / kGroup;
    ACPF_CUDA(launch_nr_newton(d, p->hs, wsb, io, tol_mismatch, max_newton, st, &nl, nr_graphs(p)));
    ACPF_CUDA(cudaEventRecord(p->tev[2 * ci + 1], st));
    launches += nl;
    if (dev_ptrs) continue;
    if (!dev_ptrs) {
      ACPF_CUDA(cudaMemcpyAsync(theta_out + s0 * d.n_bus, io.theta_out, nb * d.n_bus * 8, cudaMemcpyDeviceToHost, st));
      ACPF_CUDA(cudaMemcpyAsync(vmag_out + s0 * d.n_bus, io.vmag_out, nb * d.n_bus * 8, cudaMemcpyDeviceToHost, st));
      if (final_mismatch_inf)
        ACPF_CUDA(cudaMemcpyAsync(final_mismatch_inf + s0, io.fnorm, nb * 8, cudaMemcpyDeviceToHost, st));
      if (iterations)
        ACPF_CUDA(cudaMemcpyAsync(iterations + s0, io.iterations, nb * 4, cudaMemcpyDeviceToHost, st));
      if (status) ACPF_CUDA(cudaMemcpyAsync(status + s0, io.status, nb * 4, cudaMemcpyDeviceToHost, st));
      if (converged) ACPF_CUDA(cudaMemcpyAsync(converged + s0, io.converged, nb, cudaMemcpyDeviceToHost, st));
    }
    ACPF_CUDA(cudaEventSynchronize(p->tev[2 * ci + 1]));
    float ms = 0.0f;
    ACPF_CUDA(cudaEventElapsedTime(&ms, p->tev[2 * ci], p->tev[2 * ci + 1]));
    total_ms += ms;
  }
  if (dev_ptrs) {  // resolved lazily by acpf_nr_last_timing
    p->pending_chunks = (int)ci;
    p->pending_launches = launches;
    return ACPF_OK;
  }
  ACPF_CUDA(cudaStreamSynchronize(st));
  p->last_ms = total_ms;
  p->last_launches = launches + nr_take_device_launches(p->ws);
  return ACPF_OK;
}

acpf_status acpf_nr_last_timing(acpf_nr_plan_t p, double* kernel_ms, int32_t* launches) {
  if (!p) {
    set_error("acpf_nr_last_timing: null plan");
    return ACPF_EINVAL;
  }
  if (p->pending_chunks > 0) {  // the last solve was a device-pointer (asynchronous) one
    DeviceGuard dg(p->device);
    float total = 0.0f;
    for (int c = 0; c < p->pending_chunks; ++c) {
      float ms = 0.0f;
      ACPF_CUDA(cudaEventSynchronize(p->tev[2 * c + 1]));
      ACPF_CUDA(cudaEventElapsedTime(&ms, p->tev[2 * c], p->tev[2 * c + 1]));
      total += ms;
    }
    p->last_ms = total;
    p->last_launches = p->pending_launches + nr_take_device_launches(p->ws);
    p->pending_chunks = 0;
  }
  if (kernel_ms) *kernel_ms = p->last_ms;
  if (launches) *launches = p->last_launches;
  return ACPF_OK;
}

acpf_status acpf_nr_plan_destroy(acpf_nr_plan_t p) {
  if (!p) return ACPF_OK;
  {
    DeviceGuard dg(p->device);
    if (p->ev0) cudaEventDestroy(p->ev0);
    if (p->ev1) cudaEventDestroy(p->ev1);
    for (cudaEvent_t e : p->tev) cudaEventDestroy(e);
    for (int k = 0; k < 2; ++k) {
      if (p->ev_h2d[k]) cudaEventDestroy(p->ev_h2d[k]);
      if (p->ev_kend[k]) cudaEventDestroy(p->ev_kend[k]);
      if (p->ev_d2h[k]) cudaEventDestroy(p->ev_d2h[k]);
    }
    if (p->copy_stream) cudaStreamDestroy(p->copy_stream);
    p->graphs.release();
    if (p->graphs.capture) cudaStreamDestroy(p->graphs.capture);
    if (p->host_active) cudaFreeHost(p->host_active);
    for (NrLane& L : p->lanes) {
      L.graphs.release();
      if (L.graphs.capture) cudaStreamDestroy(L.graphs.capture);
      if (L.st) cudaStreamDestroy(L.st);
      if (L.cs_in) cudaStreamDestroy(L.cs_in);
      if (L.cs_out) cudaStreamDestroy(L.cs_out);
      for (int i = 0; i < 2; ++i) {
        if (L.ev_in[i]) cudaEventDestroy(L.ev_in[i]);
        if (L.ev_done[i]) cudaEventDestroy(L.ev_done[i]);
        if (L.ev_out[i]) cudaEventDestroy(L.ev_out[i]);
      }
      if (L.ev_h2d) cudaEventDestroy(L.ev_h2d);
      if (L.ev_end) cudaEventDestroy(L.ev_end);
      if (L.host_active) cudaFreeHost(L.host_active);
      L.work.release();
      L.stage.release();
    }
    p->work.release();
    p->stage.release();
    p->model.release();
  }
  delete p;
  return ACPF_OK;
}

// ---------------------------------------------------------------------------
// Z-Bus
// ---------------------------------------------------------------------------

acpf_status acpf_zbus_plan_create(int32_t device, int32_t n, int32_t n_l, const int32_t* l_index,
                                  const double* zl, const double* v0, int32_t n_wye,
                                  const int32_t* wye_idx, int32_t n_delta, const int32_t* delta_p,
                                  const int32_t* delta_q, double voltage_floor,
                                  acpf_zbus_plan_t* out) {
  if (!out || n <= 0 || n_l < 0 || (n_l && (!l_index || !zl)) || !v0 || n_wye < 0 ||
      n_delta < 0 || (n_wye && !wye_idx) || (n_delta && (!delta_p || !delta_q)) ||
      n_l > 1024) {
    set_error("acpf_zbus_plan_create: invalid argument");
    return ACPF_EINVAL;
  }
  *out = nullptr;
  std::vector<int32_t> lpos(n, -1);
  for (int k = 0; k < n_l; ++k) {
    if (l_index[k] < 0 || l_index[k] >= n || (k && l_index[k] <= l_index[k - 1])) {
      set_error("acpf_zbus_plan_create: l_index must be sorted, unique, in range");
      return ACPF_EINVAL;
    }
    lpos[l_index[k]] = k;
  }
  auto map = [&](const int32_t* idx, int cnt, std::vector<int32_t>& o) -> bool {
    o.resize(cnt);
    for (int k = 0; k < cnt; ++k) {
      if (idx[k] < 0 || idx[k] >= n || lpos[idx[k]] < 0) return false;
      o[k] = lpos[idx[k]];
    }
    return true;
  };
  std::vector<int32_t> wl, dpl, dql;
  if (!map(wye_idx, n_wye, wl) || !map(delta_p, n_delta, dpl) || !map(delta_q, n_delta, dql)) {
    set_error("acpf_zbus_plan_create: load index not in l_index");
    return ACPF_EINVAL;
  }
  acpf_zbus_plan* p = new (std::nothrow) acpf_zbus_plan();
  if (!p) {
    set_error("host allocation failed");
    return ACPF_ENOMEM;
  }
  p->device = device;
  DeviceGuard dg(device);
  p->h_wye.assign(wye_idx, wye_idx + n_wye);
  p->h_dp.assign(delta_p, delta_p + n_delta);
  p->h_dq.assign(delta_q, delta_q + n_delta);
  p->floor = voltage_floor;
  p->n_wye = n_wye;
  p->n_delta = n_delta;
  ZbDeviceModel& d = p->dm;
  d.n = n;
  d.n_l = n_l;
  d.kpad = std::max(4, ((n_l + 3) / 4) * 4);
  d.n_rb = (n + kZbRows - 1) / kZbRows;
  d.n_wye = n_wye;
  d.n_delta = n_delta;
  d.floor = voltage_floor;
  std::vector<double> frag(zbus_frag_doubles(d.n_rb, d.kpad));
  zbus_pack_fragments(zl, n, n_l, d.n_rb, d.kpad, frag.data());
  std::vector<double2> v0p((size_t)d.n_rb * kZbRows, make_double2(0.0, 0.0));
  for (int r = 0; r < n; ++r) v0p[r] = make_double2(v0[2 * r], v0[2 * r + 1]);
  std::vector<int32_t> lrow(l_index, l_index + n_l);
  cudaError_t e = cudaSuccess;
  auto up = [&](auto** dst, const auto* src, size_t cnt) {
    if (e == cudaSuccess) e = p->model.upload(dst, src, cnt);
  };
  up(const_cast<double**>(&d.zfrag), frag.data(), frag.size());
  up(const_cast<double2**>(&d.v0), v0p.data(), v0p.size());
  up(const_cast<int32_t**>(&d.l_row), lrow.data(), lrow.size());
  up(const_cast<int32_t**>(&d.wye_l), wl.data(), wl.size());
  up(const_cast<int32_t**>(&d.dp_l), dpl.data(), dpl.size());
  up(const_cast<int32_t**>(&d.dq_l), dql.data(), dql.size());
  d.lpos_of_row = nullptr;
  double* mag0_dev = nullptr;
  if (e == cudaSuccess) e = p->model.upload(&mag0_dev, (const double*)nullptr, 0);
  if (e == cudaSuccess) e = cudaEventCreate(&p->ev0);
  if (e == cudaSuccess) e = cudaEventCreate(&p->ev1);
  if (e == cudaSuccess) {
    ZbBatchIO io{};
    e = launch_zbus(d, io, 0.0, 1, true, mag0_dev, nullptr, 0);
  }
  if (e == cudaSuccess) e = cudaMemcpy(&d.mag0, mag0_dev, 8, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) {
    set_error(std::string("acpf_zbus_plan_create: ") + cudaGetErrorString(e));
    delete p;
    return e == cudaErrorMemoryAllocation ? ACPF_ENOMEM : ACPF_ECUDA;
  }
  *out = p;
  return ACPF_OK;
}

static acpf_status zbus_solve_host(acpf_zbus_plan* p, int64_t batch, const double* s_wye,
                                   const double* s_delta, double tol, int32_t max_iter, double* v_out,
                                   uint8_t* converged, int32_t* iterations, double* final_delta,
                                   double* residual_inf, int32_t* status, int32_t* floor_slot,
                                   cudaStream_t st) {
  // Two staging sets; chunk c+1's H2D and chunk c's D2H run on a copy stream
  // while chunk c+1 computes, so the voltage read-back overlaps the solve.
  const ZbDeviceModel& d = p->dm;
  const int64_t chunk = std::min<int64_t>(batch, std::max<int64_t>(1, env_int("ACPF_ZBUS_CHUNK", 16384)));
  const size_t in_b = (size_t)(d.n_wye + d.n_delta) * 16;
  const size_t out_b = (size_t)d.n * 16 + 1 + 4 + 8 + 8 + 4 + 4;
  // each staging set (and every buffer inside it) starts on a 256-byte
  // boundary: the kernels read s_wye/s_delta/v as double2
  const size_t set_b = (((size_t)chunk * (in_b + out_b) + 8 * 256) + 255) & ~(size_t)255;
  acpf_status rc = ensure_stage(p->stage, p->stage_bytes, p->stage_base, 2 * set_b);
  if (rc != ACPF_OK) return rc;
  if (!p->copy_stream) ACPF_CUDA(cudaStreamCreateWithFlags(&p->copy_stream, cudaStreamNonBlocking));
  for (int k = 0; k < 2; ++k) {
    if (!p->ev_h2d[k]) ACPF_CUDA(cudaEventCreateWithFlags(&p->ev_h2d[k], cudaEventDisableTiming));
    if (!p->ev_kend[k]) ACPF_CUDA(cudaEventCreateWithFlags(&p->ev_kend[k], cudaEventDisableTiming));
    if (!p->ev_d2h[k]) ACPF_CUDA(cudaEventCreateWithFlags(&p->ev_d2h[k], cudaEventDisableTiming));
  }
  cudaStream_t cs = p->copy_stream;
  const int64_t nchunks = (batch + chunk - 1) / chunk;
  struct Set {
    double2 *sw, *sd, *vo;
    double *fd, *rs;
    int32_t *it, *stt, *fs;
    uint8_t* cv;
  } sets[2];
  for (int k = 0; k < 2; ++k) {
    char* b = (char*)p->stage_base + k * set_b;
    auto take = [&](size_t bytes) {
      char* r = b;
      b += (bytes + 255) & ~(size_t)255;
      return r;
    };
    Set& S = sets[k];
    S.sw = (double2*)take((size_t)chunk * d.n_wye * 16);
    S.sd = (double2*)take((size_t)chunk * d.n_delta * 16);
    S.vo = (double2*)take((size_t)chunk * d.n * 16);
    S.fd = (double*)take((size_t)chunk * 8);
    S.rs = (double*)take((size_t)chunk * 8);
    S.it = (int32_t*)take((size_t)chunk * 4);
    S.stt = (int32_t*)take((size_t)chunk * 4);
    S.fs = (int32_t*)take((size_t)chunk * 4);
    S.cv = (uint8_t*)take((size_t)chunk);
  }
  std::vector<cudaEvent_t> tev(2 * nchunks, nullptr);
  for (auto& e : tev) ACPF_CUDA(cudaEventCreate(&e));
  auto h2d = [&](int64_t c) -> acpf_status {
    const int k = (int)(c & 1);
    const int64_t s0 = c * chunk, nb = std::min(chunk, batch - s0);
    ACPF_CUDA(cudaStreamWaitEvent(cs, p->ev_kend[k], 0));  // inputs of chunk c-2 consumed
    if (d.n_wye)
      ACPF_CUDA(cudaMemcpyAsync(sets[k].sw, s_wye + 2 * s0 * d.n_wye, nb * d.n_wye * 16, cudaMemcpyHostToDevice, cs));
    if (d.n_delta)
      ACPF_CUDA(cudaMemcpyAsync(sets[k].sd, s_delta + 2 * s0 * d.n_delta, nb * d.n_delta * 16, cudaMemcpyHostToDevice, cs));
    ACPF_CUDA(cudaEventRecord(p->ev_h2d[k], cs));
    return ACPF_OK;
  };
  int launches = 0;
  if ((rc = h2d(0)) != ACPF_OK) return rc;
  for (int64_t c = 0; c < nchunks; ++c) {
    const int k = (int)(c & 1);
    const int64_t s0 = c * chunk, nb = std::min(chunk, batch - s0);
    const Set& S = sets[k];
    ZbBatchIO io{};
    io.batch = nb;
    io.s_wye = S.sw;
    io.s_delta = S.sd;
    io.v_out = S.vo;
    io.final_delta = S.fd;
    io.residual = S.rs;
    io.iterations = S.it;
    io.status = S.stt;
    io.floor_slot = S.fs;
    io.converged = S.cv;
    ACPF_CUDA(cudaStreamWaitEvent(st, p->ev_h2d[k], 0));
    if (c >= 2) ACPF_CUDA(cudaStreamWaitEvent(st, p->ev_d2h[k], 0));  // outputs of chunk c-2 read back
    int nl = 0;
    ACPF_CUDA(cudaEventRecord(tev[2 * c], st));
    ACPF_CUDA(launch_zbus(d, io, tol, max_iter, false, nullptr, &nl, st));
    ACPF_CUDA(cudaEventRecord(tev[2 * c + 1], st));
    ACPF_CUDA(cudaEventRecord(p->ev_kend[k], st));
    launches += nl;
    if (c + 1 < nchunks && (rc = h2d(c + 1)) != ACPF_OK) return rc;
    ACPF_CUDA(cudaStreamWaitEvent(cs, p->ev_kend[k], 0));
    ACPF_CUDA(cudaMemcpyAsync(v_out + 2 * s0 * d.n, S.vo, nb * d.n * 16, cudaMemcpyDeviceToHost, cs));
    if (converged) ACPF_CUDA(cudaMemcpyAsync(converged + s0, S.cv, nb, cudaMemcpyDeviceToHost, cs));
    if (iterations) ACPF_CUDA(cudaMemcpyAsync(iterations + s0, S.it, nb * 4, cudaMemcpyDeviceToHost, cs));
    if (final_delta) ACPF_CUDA(cudaMemcpyAsync(final_delta + s0, S.fd, nb * 8, cudaMemcpyDeviceToHost, cs));
    if (residual_inf) ACPF_CUDA(cudaMemcpyAsync(residual_inf + s0, S.rs, nb * 8, cudaMemcpyDeviceToHost, cs));
    if (status) ACPF_CUDA(cudaMemcpyAsync(status + s0, S.stt, nb * 4, cudaMemcpyDeviceToHost, cs));
    if (floor_slot) ACPF_CUDA(cudaMemcpyAsync(floor_slot + s0, S.fs, nb * 4, cudaMemcpyDeviceToHost, cs));
    ACPF_CUDA(cudaEventRecord(p->ev_d2h[k], cs));
  }
  ACPF_CUDA(cudaStreamSynchronize(cs));
  ACPF_CUDA(cudaStreamSynchronize(st));
  float total = 0.0f;
  for (int64_t c = 0; c < nchunks; ++c) {
    float ms = 0.0f;
    ACPF_CUDA(cudaEventElapsedTime(&ms, tev[2 * c], tev[2 * c + 1]));
    total += ms;
  }
  for (auto& e : tev) cudaEventDestroy(e);
  p->last_ms = total;
  p->last_launches = launches;
  return ACPF_OK;
}

acpf_status acpf_zbus_solve(acpf_zbus_plan_t p, int64_t batch, const double* s_wye,
                            const double* s_delta, double tol, int32_t max_iter, double* v_out,
                            uint8_t* converged, int32_t* iterations, double* final_delta,
                            double* residual_inf, int32_t* status, int32_t* floor_slot,
                            uint32_t flags, void* cuda_stream) {
  const ZbDeviceModel& d = p ? p->dm : ZbDeviceModel{};
  if (!p || batch < 0 || !v_out || max_iter < 1 || !(tol > 0) || (d.n_wye && !s_wye) ||
      (d.n_delta && !s_delta) || flags > 1u) {
    set_error("acpf_zbus_solve: invalid argument");
    return ACPF_EINVAL;
  }
  if (batch == 0) return ACPF_OK;
  DeviceGuard dg(p->device);
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const bool dev_ptrs = flags & ACPF_DEVICE_PTRS;
  if (!dev_ptrs)
    return zbus_solve_host(p, batch, s_wye, s_delta, tol, max_iter, v_out, converged, iterations,
                           final_delta, residual_inf, status, floor_slot, st);
  int64_t chunk = batch;
  const size_t in_b = (size_t)(d.n_wye + d.n_delta) * 16;
  const size_t out_b = (size_t)d.n * 16 + 1 + 4 + 8 + 8 + 4 + 4;
  if (!dev_ptrs) {
    acpf_status rc = ensure_stage(p->stage, p->stage_bytes, p->stage_base, (size_t)chunk * (in_b + out_b) + 256);
    if (rc != ACPF_OK) return rc;
  }
  float total_ms = 0.0f;
  int launches = 0;
  for (int64_t s0 = 0; s0 < batch; s0 += chunk) {
    const int64_t nb = std::min(chunk, batch - s0);
    ZbBatchIO io{};
    io.batch = nb;
    if (dev_ptrs) {
      io.s_wye = (const double2*)(s_wye ? s_wye + 2 * s0 * d.n_wye : nullptr);
      io.s_delta = (const double2*)(s_delta ? s_delta + 2 * s0 * d.n_delta : nullptr);
      io.v_out = (double2*)(v_out + 2 * s0 * d.n);
      io.converged = converged ? converged + s0 : nullptr;
      io.iterations = iterations ? iterations + s0 : nullptr;
      io.final_delta = final_delta ? final_delta + s0 : nullptr;
      io.residual = residual_inf ? residual_inf + s0 : nullptr;
      io.status = status ? status + s0 : nullptr;
      io.floor_slot = floor_slot ? floor_slot + s0 : nullptr;
    } else {
      char* b = (char*)p->stage_base;
      double2* sw = (double2*)b;
      b += (size_t)chunk * d.n_wye * 16;
      double2* sd = (double2*)b;
      b += (size_t)chunk * d.n_delta * 16;
      double2* vo = (double2*)b;
      b += (size_t)chunk * d.n * 16;
      double* fd = (double*)b;
      b += (size_t)chunk * 8;
      double* rs = (double*)b;
      b += (size_t)chunk * 8;
      int32_t* it = (int32_t*)b;
      b += (size_t)chunk * 4;
      int32_t* stt = (int32_t*)b;
      b += (size_t)chunk * 4;
      int32_t* fs = (int32_t*)b;
      b += (size_t)chunk * 4;
      uint8_t* cv = (uint8_t*)b;
      if (d.n_wye)
        ACPF_CUDA(cudaMemcpyAsync(sw, s_wye + 2 * s0 * d.n_wye, nb * d.n_wye * 16, cudaMemcpyHostToDevice, st));
      if (d.n_delta)
        ACPF_CUDA(cudaMemcpyAsync(sd, s_delta + 2 * s0 * d.n_delta, nb * d.n_delta * 16, cudaMemcpyHostToDevice, st));
      io.s_wye = sw;
      io.s_delta = sd;
      io.v_out = vo;
      io.final_delta = fd;
      io.residual = rs;
      io.iterations = it;
      io.status = stt;
      io.floor_slot = fs;
      io.converged = cv;
    }
    int nl = 0;
    ACPF_CUDA(cudaEventRecord(p->ev0, st));
    ACPF_CUDA(launch_zbus(d, io, tol, max_iter, false, nullptr, &nl, st));
    ACPF_CUDA(cudaEventRecord(p->ev1, st));
    launches += nl;
    if (dev_ptrs) {  // one launch, asynchronous: resolved by acpf_zbus_last_timing
      p->pending = true;
      p->last_launches = launches;
      return ACPF_OK;
    }
    if (!dev_ptrs) {
      ACPF_CUDA(cudaMemcpyAsync(v_out + 2 * s0 * d.n, io.v_out, nb * d.n * 16, cudaMemcpyDeviceToHost, st));
      if (converged) ACPF_CUDA(cudaMemcpyAsync(converged + s0, io.converged, nb, cudaMemcpyDeviceToHost, st));
      if (iterations) ACPF_CUDA(cudaMemcpyAsync(iterations + s0, io.iterations, nb * 4, cudaMemcpyDeviceToHost, st));
      if (final_delta) ACPF_CUDA(cudaMemcpyAsync(final_delta + s0, io.final_delta, nb * 8, cudaMemcpyDeviceToHost, st));
      if (residual_inf) ACPF_CUDA(cudaMemcpyAsync(residual_inf + s0, io.residual, nb * 8, cudaMemcpyDeviceToHost, st));
      if (status) ACPF_CUDA(cudaMemcpyAsync(status + s0, io.status, nb * 4, cudaMemcpyDeviceToHost, st));
      if (floor_slot) ACPF_CUDA(cudaMemcpyAsync(floor_slot + s0, io.floor_slot, nb * 4, cudaMemcpyDeviceToHost, st));
    }
    ACPF_CUDA(cudaEventSynchronize(p->ev1));
    float ms = 0.0f;
    ACPF_CUDA(cudaEventElapsedTime(&ms, p->ev0, p->ev1));
    total_ms += ms;
  }
  ACPF_CUDA(cudaStreamSynchronize(st));
  p->last_ms = total_ms;
  p->last_launches = launches;
  return ACPF_OK;
}

acpf_status acpf_zbus_last_timing(acpf_zbus_plan_t p, double* kernel_ms, int32_t* launches) {
  if (!p) {
    set_error("acpf_zbus_last_timing: null plan");
    return ACPF_EINVAL;
  }
  if (p->pending) {
    DeviceGuard dg(p->device);
    float ms = 0.0f;
    ACPF_CUDA(cudaEventSynchronize(p->ev1));
    ACPF_CUDA(cudaEventElapsedTime(&ms, p->ev0, p->ev1));
    p->last_ms = ms;
    p->pending = false;
  }
  if (kernel_ms) *kernel_ms = p->last_ms;
  if (launches) *launches = p->last_launches;
  return ACPF_OK;
}

acpf_status acpf_zbus_plan_destroy(acpf_zbus_plan_t p) {
  if (!p) return ACPF_OK;
  {
    DeviceGuard dg(p->device);
    if (p->ev0) cudaEventDestroy(p->ev0);
    if (p->ev1) cudaEventDestroy(p->ev1);
    for (int k = 0; k < 2; ++k) {
      if (p->ev_h2d[k]) cudaEventDestroy(p->ev_h2d[k]);
      if (p->ev_kend[k]) cudaEventDestroy(p->ev_kend[k]);
      if (p->ev_d2h[k]) cudaEventDestroy(p->ev_d2h[k]);
    }
    if (p->copy_stream) cudaStreamDestroy(p->copy_stream);
    p->stage.release();
    p->model.release();
  }
  delete p;
  return ACPF_OK;
}

// ---------------------------------------------------------------------------
// Seeded scenario generation
// ---------------------------------------------------------------------------

namespace {
// device staging for host-pointer outputs + small per-call uploads
struct TmpArena {
  acpf::DevArena a;
};
}  // namespace

acpf_status acpf_philox_multipliers(uint64_t seed, int64_t start, int64_t count, int32_t n_elem,
                                    double spread, double* out, uint32_t flags, void* cuda_stream) {
  if (start < 0 || count < 0 || n_elem < 0 || !out || !(spread >= 0 && spread < 1) || flags > 1u) {
    set_error("acpf_philox_multipliers: invalid argument");
    return ACPF_EINVAL;
  }
  if (count == 0 || n_elem == 0) return ACPF_OK;
  cudaStream_t st = (cudaStream_t)cuda_stream;
  TmpArena t;
  double* d = out;
  const size_t bytes = (size_t)count * n_elem * 8;
  if (!(flags & ACPF_DEVICE_PTRS)) ACPF_CUDA(t.a.alloc((void**)&d, bytes));
  ACPF_CUDA(launch_philox_multipliers(seed, start, count, n_elem, spread, d, st));
  if (!(flags & ACPF_DEVICE_PTRS)) ACPF_CUDA(cudaMemcpyAsync(out, d, bytes, cudaMemcpyDeviceToHost, st));
  ACPF_CUDA(cudaStreamSynchronize(st));
  return ACPF_OK;
}

acpf_status acpf_nr_scenarios(acpf_nr_plan_t p, uint64_t seed, int64_t start, int64_t count,
                              double spread, int32_t n_elem, const int32_t* element_bus,
                              const double* p_load, const double* q_load, const double* p_gen,
                              const double* q_gen, double* p_spec, double* q_spec, uint32_t flags,
                              void* cuda_stream) {
  if (!p || start < 0 || count < 0 || n_elem < 0 || (n_elem && !element_bus) || !p_load || !q_load ||
      !p_gen || !q_gen || !(spread >= 0 && spread < 1) || flags > 1u ||
      (p->dm.n_theta && !p_spec) || (p->dm.n_q && !q_spec)) {
    set_error("acpf_nr_scenarios: invalid argument");
    return ACPF_EINVAL;
  }
  if (count == 0) return ACPF_OK;
  DeviceGuard dg(p->device);
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const int nb = p->dm.n_bus, nt = p->dm.n_theta, nq = p->dm.n_q;
  std::vector<double> pb(nt), qb(nq);
  for (int b = 0; b < nb; ++b) {
    if (p->h_tpos[b] >= 0) pb[p->h_tpos[b]] = p_gen[b] - p_load[b];
    if (p->h_qidx[b] >= 0) qb[p->h_qidx[b]] = q_gen[b] - q_load[b];
  }
  std::vector<int32_t> et(n_elem), eq(n_elem);
  std::vector<double> epl(n_elem), eql(n_elem), epg(n_elem), eqg(n_elem);
  for (int e = 0; e < n_elem; ++e) {
    const int b = element_bus[e];
    if (b < 0 || b >= nb) {
      set_error("acpf_nr_scenarios: element bus out of range");
      return ACPF_EINVAL;
    }
    et[e] = p->h_tpos[b];
    eq[e] = p->h_qidx[b];
    epl[e] = p_load[b];
    eql[e] = q_load[b];
    epg[e] = p_gen[b];
    eqg[e] = q_gen[b];
  }
  TmpArena t;
  NrScenarioArgs a{};
  cudaError_t e = cudaSuccess;
  auto up = [&](auto** dst, const auto* src, size_t cnt) {
    if (e == cudaSuccess) e = t.a.upload(dst, src, cnt);
  };
  up(const_cast<double**>(&a.p_base), pb.data(), pb.size());
  up(const_cast<double**>(&a.q_base), qb.data(), qb.size());
  up(const_cast<int32_t**>(&a.elem_tpos), et.data(), et.size());
  up(const_cast<int32_t**>(&a.elem_qidx), eq.data(), eq.size());
  up(const_cast<double**>(&a.elem_pl), epl.data(), epl.size());
  up(const_cast<double**>(&a.elem_ql), eql.data(), eql.size());
  up(const_cast<double**>(&a.elem_pg), epg.data(), epg.size());
  up(const_cast<double**>(&a.elem_qg), eqg.data(), eqg.size());
  ACPF_CUDA(e);
  a.seed = seed;
  a.start = start;
  a.count = count;
  a.spread = spread;
  a.n_elem = n_elem;
  a.n_theta = nt;
  a.n_q = nq;
  a.p_spec = p_spec;
  a.q_spec = q_spec;
  const bool host = !(flags & ACPF_DEVICE_PTRS);
  if (host) {
    ACPF_CUDA(t.a.alloc((void**)&a.p_spec, (size_t)count * nt * 8));
    ACPF_CUDA(t.a.alloc((void**)&a.q_spec, (size_t)count * nq * 8));
  }
  ACPF_CUDA(launch_nr_scenarios(a, st));
  if (host) {
    if (nt) ACPF_CUDA(cudaMemcpyAsync(p_spec, a.p_spec, (size_t)count * nt * 8, cudaMemcpyDeviceToHost, st));
    if (nq) ACPF_CUDA(cudaMemcpyAsync(q_spec, a.q_spec, (size_t)count * nq * 8, cudaMemcpyDeviceToHost, st));
  }
  ACPF_CUDA(cudaStreamSynchronize(st));
  return ACPF_OK;
}

acpf_status acpf_zbus_scenarios(acpf_zbus_plan_t p, uint64_t seed, int64_t start, int64_t count,
                                double spread, int32_t n_elem, const int32_t* elem_target,
                                const double* wye_s, const double* delta_s, double* s_wye,
                                double* s_delta, uint32_t flags, void* cuda_stream) {
  if (!p || start < 0 || count < 0 || n_elem < 0 || (n_elem && !elem_target) ||
      (p->n_wye && (!wye_s || !s_wye)) || (p->n_delta && (!delta_s || !s_delta)) ||
      !(spread >= 0 && spread < 1) || flags > 1u || n_elem != p->n_wye + p->n_delta) {
    set_error("acpf_zbus_scenarios: invalid argument");
    return ACPF_EINVAL;
  }
  if (count == 0) return ACPF_OK;
  for (int k = 0; k < n_elem; ++k) {
    const int tg = elem_target[k];
    if ((tg >= 0 && tg >= p->n_wye) || (tg < 0 && -tg - 1 >= p->n_delta)) {
      set_error("acpf_zbus_scenarios: element target out of range");
      return ACPF_EINVAL;
    }
  }
  DeviceGuard dg(p->device);
  cudaStream_t st = (cudaStream_t)cuda_stream;
  TmpArena t;
  ZbScenarioArgs a{};
  cudaError_t e = cudaSuccess;
  e = t.a.upload(const_cast<int32_t**>(&a.elem_target), elem_target, (size_t)n_elem);
  if (e == cudaSuccess)
    e = t.a.upload(const_cast<double2**>(&a.wye_s), reinterpret_cast<const double2*>(wye_s), (size_t)p->n_wye);
  if (e == cudaSuccess)
    e = t.a.upload(const_cast<double2**>(&a.delta_s), reinterpret_cast<const double2*>(delta_s),
                   (size_t)p->n_delta);
  ACPF_CUDA(e);
  a.seed = seed;
  a.start = start;
  a.count = count;
  a.spread = spread;
  a.n_elem = n_elem;
  a.n_wye = p->n_wye;
  a.n_delta = p->n_delta;
  a.s_wye = reinterpret_cast<double2*>(s_wye);
  a.s_delta = reinterpret_cast<double2*>(s_delta);
  const bool host = !(flags & ACPF_DEVICE_PTRS);
  if (host) {
    ACPF_CUDA(t.a.alloc((void**)&a.s_wye, (size_t)count * p->n_wye * 16));
    ACPF_CUDA(t.a.alloc((void**)&a.s_delta, (size_t)count * p->n_delta * 16));
  }
  ACPF_CUDA(launch_zb_scenarios(a, st));
  if (host) {
    if (p->n_wye)
      ACPF_CUDA(cudaMemcpyAsync(s_wye, a.s_wye, (size_t)count * p->n_wye * 16, cudaMemcpyDeviceToHost, st));
    if (p->n_delta)
      ACPF_CUDA(cudaMemcpyAsync(s_delta, a.s_delta, (size_t)count * p->n_delta * 16, cudaMemcpyDeviceToHost, st));
  }
  ACPF_CUDA(cudaStreamSynchronize(st));
  return ACPF_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Certificates (kernels in cert_kernel.cu)
// ---------------------------------------------------------------------------

namespace {

// Device views of the caller's arrays: the pointers themselves for
// ACPF_DEVICE_PTRS, else device copies (inputs uploaded, outputs allocated).
struct Staged {
  DevArena a;
  cudaError_t e = cudaSuccess;
  bool host;
  cudaStream_t st;
  Staged(uint32_t flags, cudaStream_t s) : host(!(flags & ACPF_DEVICE_PTRS)), st(s) {}
  template <class T>
  T* in(const T* p, size_t count) {
    if (!host || !p || e != cudaSuccess) return const_cast<T*>(p);
    T* d = nullptr;
    e = a.alloc((void**)&d, count * sizeof(T));
    if (e == cudaSuccess && count) e = cudaMemcpyAsync(d, p, count * sizeof(T), cudaMemcpyHostToDevice, st);
    return d;
  }
  template <class T>
  T* out(T* p, size_t count) {
    if (!host || !p || e != cudaSuccess) return p;
    T* d = nullptr;
    e = a.alloc((void**)&d, count * sizeof(T));
    return d;
  }
  template <class T>
  void back(T* host_p, const T* dev_p, size_t count) {
    if (host && host_p && e == cudaSuccess && count)
      e = cudaMemcpyAsync(host_p, dev_p, count * sizeof(T), cudaMemcpyDeviceToHost, st);
  }
};

}  // namespace

extern "C" {

acpf_status acpf_nr_plan_set_branches(acpf_nr_plan_t p, int32_t n_br, const int32_t* from_bus,
                                      const int32_t* to_bus, const double* y4, const double* bus_gs) {
  if (!p || n_br < 0 || (n_br && (!from_bus || !to_bus || !y4)) || !bus_gs) {
    set_error("acpf_nr_plan_set_branches: invalid argument");
    return ACPF_EINVAL;
  }
  const int nb = p->dm.n_bus;
  for (int b = 0; b < n_br; ++b)
    if (from_bus[b] < 0 || from_bus[b] >= nb || to_bus[b] < 0 || to_bus[b] >= nb) {
      set_error("acpf_nr_plan_set_branches: branch bus out of range");
      return ACPF_EINVAL;
    }
  if (nr_cert_smem(nb) > 227 * 1024) {
    set_error("acpf_nr_plan_set_branches: network too large for the certificate kernel");
    return ACPF_ESTRUCT;
  }
  DeviceGuard dg(p->device);
  p->cert_arena.release();
  NrCertModel c{};
  c.n_bus = nb;
  c.n_theta = p->dm.n_theta;
  c.n_q = p->dm.n_q;
  c.n_br = n_br;
  c.y_rowptr = p->dm.y_rowptr;
  c.y_col = p->dm.y_col;
  c.y_val = p->dm.y_val;
  c.tpos = p->dm.tpos;
  c.qidx = p->dm.qidx;
  cudaError_t e = cudaSuccess;
  auto up = [&](auto** dst, const auto* src, size_t cnt) {
    if (e == cudaSuccess) e = p->cert_arena.upload(dst, src, cnt);
  };
  up(const_cast<int32_t**>(&c.br_f), from_bus, (size_t)n_br);
  up(const_cast<int32_t**>(&c.br_t), to_bus, (size_t)n_br);
  up(const_cast<double2**>(&c.br_y), reinterpret_cast<const double2*>(y4), (size_t)n_br * 4);
  up(const_cast<double**>(&c.gs), bus_gs, (size_t)nb);
  ACPF_CUDA(e);
  p->cert = c;
  return ACPF_OK;
}

acpf_status acpf_nr_certify(acpf_nr_plan_t p, int64_t batch, const double* theta, const double* vmag,
                            const double* p_spec, const double* q_spec, double* mismatch_inf,
                            double* slack_balance, double* branch_loss, uint32_t flags, void* cuda_stream) {
  if (!p || batch < 0 || flags > 1u || (batch && (!theta || !vmag)) ||
      (batch && p->dm.n_theta && !p_spec) || (batch && p->dm.n_q && !q_spec)) {
    set_error("acpf_nr_certify: invalid argument");
    return ACPF_EINVAL;
  }
  if (p->cert.n_br < 0) {
    set_error("acpf_nr_certify: call acpf_nr_plan_set_branches first");
    return ACPF_EINVAL;
  }
  if (batch == 0) return ACPF_OK;
  DeviceGuard dg(p->device);
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const size_t nb = p->dm.n_bus, nt = p->dm.n_theta, nq = p->dm.n_q, B = (size_t)batch;
  Staged g(flags, st);
  NrCertIO io{};
  io.batch = batch;
  io.theta = g.in(theta, B * nb);
  io.vmag = g.in(vmag, B * nb);
  io.p_spec = g.in(p_spec, B * nt);
  io.q_spec = g.in(q_spec, B * nq);
  io.mismatch_inf = g.out(mismatch_inf, B);
  io.slack_balance = g.out(slack_balance, B);
  io.branch_loss = g.out(branch_loss, B);
  ACPF_CUDA(g.e);
  ACPF_CUDA(launch_nr_cert(p->cert, io, st));
  g.back(mismatch_inf, io.mismatch_inf, B);
  g.back(slack_balance, io.slack_balance, B);
  g.back(branch_loss, io.branch_loss, B);
  ACPF_CUDA(g.e);
  ACPF_CUDA(cudaStreamSynchronize(st));
  return ACPF_OK;
}

acpf_status acpf_zbus_plan_set_network(acpf_zbus_plan_t p, const int32_t* ynn_rowptr, const int32_t* ynn_col,
                                       const double* ynn_val, const double* inj) {
  if (!p || !ynn_rowptr || !inj) {
    set_error("acpf_zbus_plan_set_network: invalid argument");
    return ACPF_EINVAL;
  }
  const int n = p->dm.n;
  const int64_t nnz = ynn_rowptr[n];
  if (ynn_rowptr[0] != 0 || nnz < 0 || (nnz && (!ynn_col || !ynn_val))) {
    set_error("acpf_zbus_plan_set_network: bad CSR");
    return ACPF_EINVAL;
  }
  for (int k = 0; k < n; ++k)
    if (ynn_rowptr[k + 1] < ynn_rowptr[k]) {
      set_error("acpf_zbus_plan_set_network: bad CSR row pointers");
      return ACPF_EINVAL;
    }
  for (int64_t e = 0; e < nnz; ++e)
    if (ynn_col[e] < 0 || ynn_col[e] >= n) {
      set_error("acpf_zbus_plan_set_network: column out of range");
      return ACPF_EINVAL;
    }
  if (zb_cert_smem(n) > 227 * 1024) {
    set_error("acpf_zbus_plan_set_network: feeder too large for the certificate kernel");
    return ACPF_ESTRUCT;
  }
  DeviceGuard dg(p->device);
  p->cert_arena.release();
  ZbCertModel c{};
  c.n = n;
  c.n_wye = p->n_wye;
  c.n_delta = p->n_delta;
  c.floor = p->floor;
  cudaError_t e = cudaSuccess;
  auto up = [&](auto** dst, const auto* src, size_t cnt) {
    if (e == cudaSuccess) e = p->cert_arena.upload(dst, src, cnt);
  };
  up(const_cast<int32_t**>(&c.rowptr), ynn_rowptr, (size_t)n + 1);
  up(const_cast<int32_t**>(&c.col), ynn_col, (size_t)nnz);
  up(const_cast<double2**>(&c.val), reinterpret_cast<const double2*>(ynn_val), (size_t)nnz);
  up(const_cast<double2**>(&c.inj), reinterpret_cast<const double2*>(inj), (size_t)n);
  up(const_cast<int32_t**>(&c.wye_row), p->h_wye.data(), p->h_wye.size());
  up(const_cast<int32_t**>(&c.dp_row), p->h_dp.data(), p->h_dp.size());
  up(const_cast<int32_t**>(&c.dq_row), p->h_dq.data(), p->h_dq.size());
  ACPF_CUDA(e);
  p->cert = c;
  return ACPF_OK;
}

acpf_status acpf_zbus_kirchhoff(acpf_zbus_plan_t p, int64_t batch, const double* v, const double* s_wye,
                                const double* s_delta, double* kcl, uint32_t flags, void* cuda_stream) {
  if (!p || batch < 0 || flags > 1u || (batch && (!v || !kcl)) || (batch && p->n_wye && !s_wye) ||
      (batch && p->n_delta && !s_delta)) {
    set_error("acpf_zbus_kirchhoff: invalid argument");
    return ACPF_EINVAL;
  }
  if (!p->cert.rowptr) {
    set_error("acpf_zbus_kirchhoff: call acpf_zbus_plan_set_network first");
    return ACPF_EINVAL;
  }
  if (batch == 0) return ACPF_OK;
  DeviceGuard dg(p->device);
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const size_t B = (size_t)batch, n = p->dm.n;
  Staged g(flags, st);
  ZbCertIO io{};
  io.batch = batch;
  io.v = g.in(reinterpret_cast<const double2*>(v), B * n);
  io.s_wye = g.in(reinterpret_cast<const double2*>(s_wye), B * p->n_wye);
  io.s_delta = g.in(reinterpret_cast<const double2*>(s_delta), B * p->n_delta);
  io.kcl = g.out(kcl, B);
  ACPF_CUDA(g.e);
  ACPF_CUDA(launch_zb_kcl(p->cert, io, st));
  g.back(kcl, io.kcl, B);
  ACPF_CUDA(g.e);
  ACPF_CUDA(cudaStreamSynchronize(st));
  return ACPF_OK;
}

acpf_status acpf_zbus_reduce(int32_t device, int32_t n, const int32_t* ynn_rowptr, const int32_t* ynn_col,
                             const double* ynn_val, const double* rhs0, int32_t n_l, const int32_t* l_index,
                             double* zl_out, double* v0_out) {
  if (n <= 0 || !ynn_rowptr || !rhs0 || n_l < 0 || (n_l && (!l_index || !zl_out)) || !v0_out ||
      ynn_rowptr[0] != 0 || (ynn_rowptr[n] > 0 && (!ynn_col || !ynn_val))) {
    set_error("acpf_zbus_reduce: invalid argument");
    return ACPF_EINVAL;
  }
  for (int k = 0; k < n; ++k)
    if (ynn_rowptr[k + 1] < ynn_rowptr[k]) {
      set_error("acpf_zbus_reduce: bad CSR row pointers");
      return ACPF_EINVAL;
    }
  for (int64_t e = 0; e < ynn_rowptr[n]; ++e)
    if (ynn_col[e] < 0 || ynn_col[e] >= n) {
      set_error("acpf_zbus_reduce: column out of range");
      return ACPF_EINVAL;
    }
  for (int k = 0; k < n_l; ++k)
    if (l_index[k] < 0 || l_index[k] >= n) {
      set_error("acpf_zbus_reduce: l_index out of range");
      return ACPF_EINVAL;
    }
  DeviceGuard dg(device);
  return zbus_reduce_device(device, n, ynn_rowptr, ynn_col, ynn_val, rhs0, n_l, l_index, zl_out, v0_out, nullptr);
}

// ---------------------------------------------------------------------------
// GMRES-FD Newton ablation (kernels in gmres_kernel.cu)
// ---------------------------------------------------------------------------

acpf_status acpf_nr_plan_set_fd(acpf_nr_plan_t p, const double* bprime_inv, const double* bdprime_inv,
                                const int32_t* g_rowptr, const int32_t* g_col, const double* g_val) {
  if (!p || (p->dm.n_theta && !bprime_inv) || (p->dm.n_q && (!bdprime_inv || !g_rowptr))) {
    set_error("acpf_nr_plan_set_fd: invalid argument");
    return ACPF_EINVAL;
  }
  const int nt = p->dm.n_theta, nq = p->dm.n_q, nb = p->dm.n_bus;
  const int64_t gnnz = nq ? g_rowptr[nq] : 0;
  for (int64_t e = 0; e < gnnz; ++e)
    if (g_col[e] < 0 || g_col[e] >= nt) {
      set_error("acpf_nr_plan_set_fd: G column out of range");
      return ACPF_EINVAL;
    }
  std::vector<int32_t> tb(nt), qb(nq);
  for (int b = 0; b < nb; ++b) {
    if (p->h_tpos[b] >= 0) tb[p->h_tpos[b]] = b;
    if (p->h_qidx[b] >= 0) qb[p->h_qidx[b]] = b;
  }
  DeviceGuard dg(p->device);
  p->gm_arena.release();
  GmModel g{};
  g.n_bus = nb;
  g.n_theta = nt;
  g.n_q = nq;
  g.nj = nt + nq;
  g.y_rowptr = p->dm.y_rowptr;
  g.y_col = p->dm.y_col;
  g.y_val = p->dm.y_val;
  g.tpos = p->dm.tpos;
  g.qidx = p->dm.qidx;
  g.theta_init = p->dm.theta_init;
  g.vmag_init = p->dm.vmag_init;
  const std::vector<int32_t> zero_rp(nq + 1, 0);
  cudaError_t e = cudaSuccess;
  auto up = [&](auto** dst, const auto* src, size_t cnt) {
    if (e == cudaSuccess) e = p->gm_arena.upload(dst, src, cnt);
  };
  up(const_cast<int32_t**>(&g.theta_block), tb.data(), tb.size());
  up(const_cast<int32_t**>(&g.q_block), qb.data(), qb.size());
  up(const_cast<double**>(&g.binv1), bprime_inv, (size_t)nt * nt);
  up(const_cast<double**>(&g.binv2), bdprime_inv, (size_t)nq * nq);
  up(const_cast<int32_t**>(&g.g_rowptr), nq ? g_rowptr : zero_rp.data(), (size_t)nq + 1);
  up(const_cast<int32_t**>(&g.g_col), g_col, (size_t)gnnz);
  up(const_cast<double**>(&g.g_val), g_val, (size_t)gnnz);
  ACPF_CUDA(e);
  p->gm = g;
  return ACPF_OK;
}

acpf_status acpf_nr_solve_gmres(acpf_nr_plan_t p, int64_t batch, const double* p_spec, const double* q_spec,
                                double tol_mismatch, int32_t max_newton, double gmres_tol, int32_t restart,
                                int32_t max_outer, int32_t precond, double* theta_out, double* vmag_out,
                                uint8_t* converged, int32_t* iterations, double* final_mismatch_inf,
                                int32_t* status, int32_t* gmres_steps, int32_t* gmres_diag, int32_t* gmres_diag_k,
                                double* gmres_diag_relres, uint32_t flags, void* cuda_stream) {
  if (!p || batch < 0 || !theta_out || !vmag_out || max_newton < 1 || !(tol_mismatch > 0) ||
      !(gmres_tol > 0) || restart < 1 || max_outer < 1 || (precond != 0 && precond != 1) || flags > 1u ||
      (p->dm.n_theta && !p_spec) || (p->dm.n_q && !q_spec)) {
    set_error("acpf_nr_solve_gmres: invalid argument");
    return ACPF_EINVAL;
  }
  if (!p->gm.theta_block && p->dm.n_theta) {
    set_error("acpf_nr_solve_gmres: call acpf_nr_plan_set_fd first");
    return ACPF_EINVAL;
  }
  if (batch == 0) return ACPF_OK;
  DeviceGuard dg(p->device);
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const GmModel& m = p->gm;
  const int mm = std::min<int>(restart, std::max(1, m.nj));  // m = min(restart, n) (sparse.py:262)
  const int bc = (int)std::min<int64_t>(batch, std::max<int64_t>(32, env_int("ACPF_GMRES_CHUNK", 4096)));
  // workspace for one chunk
  const size_t nd = gmres_work_doubles(m, bc, mm);
  const size_t ni = (size_t)bc * (16 + (max_newton + 1)) + 8;
  DevArena wa;
  double* dbase = nullptr;
  int* ibase = nullptr;
  ACPF_CUDA(wa.alloc((void**)&dbase, nd * sizeof(double)));
  ACPF_CUDA(wa.alloc((void**)&ibase, ni * sizeof(int)));
  ACPF_CUDA(cudaMemsetAsync(ibase, 0, ni * sizeof(int), st));
  GmWork w{};
  w.bc = bc;
  {
    double* d = dbase;
    const size_t B = bc, nb = m.n_bus, nj = m.nj;
    auto take = [&](size_t n) {
      double* r = d;
      d += n;
      return r;
    };
    w.th = take(B * nb);
    w.vm = take(B * nb);
    w.u = (double2*)take(2 * B * nb);
    w.ph = (double2*)take(2 * B * nb);
    w.ic = (double2*)take(2 * B * nb);
    w.du = (double2*)take(2 * B * nb);
    w.b = take(B * nj);
    w.x = take(B * nj);
    w.wv = take(B * nj);
    w.t1 = take(B * nj);
    w.t2 = take(B * nj);
    w.vb = take(B * nj * (mm + 1));
    w.h = take(B * (size_t)(mm + 1) * mm);
    w.cs = take(B * mm);
    w.sn = take(B * mm);
    w.g = take(B * (mm + 1));
    w.y = take(B * (mm + 1));
    w.part = take(B * ((nj + 63) / 64));
    w.beta0 = take(B);
    w.beta = take(B);
    w.relres = take(B);
    w.scal = take(B);
    w.fout = take(B);
    w.gdiag_rel = take(B);
    w.fmax_bits = (unsigned long long*)take(B);
    int* q = ibase;
    auto takei = [&](size_t n) {
      int* r = q;
      q += n;
      return r;
    };
    w.flags = takei(B);
    w.nactive = takei(B);
    w.status = takei(B);
    w.iters = takei(B);
    w.gstate = takei(B);
    w.cyc = takei(B);
    w.kk = takei(B);
    w.brk = takei(B);
    w.gsum = takei(B);
    w.gtotal = takei(B);
    w.gdiag = takei(B);
    w.gdiag_k = takei(B);
    w.gsteps = takei(B * (max_newton + 1));
    w.count = takei(1);
  }
  struct PinnedInt {  // released on every return path
    int* p = nullptr;
    ~PinnedInt() {
      if (p) cudaFreeHost(p);
    }
  } host_count;
  ACPF_CUDA(cudaMallocHost((void**)&host_count.p, sizeof(int)));
  w.host_count = host_count.p;
  const bool dev_ptrs = flags & ACPF_DEVICE_PTRS;
  const size_t nt = m.n_theta, nq = m.n_q, nbus = m.n_bus;
  // device staging for host pointers (one chunk)
  double *sp = nullptr, *sq = nullptr, *sth = nullptr, *svm = nullptr, *sfn = nullptr, *sdr = nullptr;
  int32_t *sit = nullptr, *sst = nullptr, *sgs = nullptr, *sgd = nullptr, *sgk = nullptr;
  uint8_t* scv = nullptr;
  if (!dev_ptrs) {
    ACPF_CUDA(wa.alloc((void**)&sp, (size_t)bc * nt * 8 + 8));
    ACPF_CUDA(wa.alloc((void**)&sq, (size_t)bc * nq * 8 + 8));
    ACPF_CUDA(wa.alloc((void**)&sth, (size_t)bc * nbus * 8));
    ACPF_CUDA(wa.alloc((void**)&svm, (size_t)bc * nbus * 8));
    ACPF_CUDA(wa.alloc((void**)&sfn, (size_t)bc * 8));
    ACPF_CUDA(wa.alloc((void**)&sdr, (size_t)bc * 8));
    ACPF_CUDA(wa.alloc((void**)&sit, (size_t)bc * 4));
    ACPF_CUDA(wa.alloc((void**)&sst, (size_t)bc * 4));
    ACPF_CUDA(wa.alloc((void**)&sgs, (size_t)bc * max_newton * 4));
    ACPF_CUDA(wa.alloc((void**)&sgd, (size_t)bc * 4));
    ACPF_CUDA(wa.alloc((void**)&sgk, (size_t)bc * 4));
    ACPF_CUDA(wa.alloc((void**)&scv, (size_t)bc));
  }
  ACPF_CUDA(cudaEventRecord(p->ev0, st));
  cudaError_t err = cudaSuccess;
  for (int64_t s0 = 0; s0 < batch && err == cudaSuccess; s0 += bc) {
    const int64_t nb = std::min<int64_t>(bc, batch - s0);
    if (dev_ptrs) {
      w.p_spec = p_spec ? p_spec + s0 * nt : nullptr;
      w.q_spec = q_spec ? q_spec + s0 * nq : nullptr;
    } else {
      if (nt) err = cudaMemcpyAsync(sp, p_spec + s0 * nt, nb * nt * 8, cudaMemcpyHostToDevice, st);
      if (nq && err == cudaSuccess) err = cudaMemcpyAsync(sq, q_spec + s0 * nq, nb * nq * 8, cudaMemcpyHostToDevice, st);
      w.p_spec = sp;
      w.q_spec = sq;
    }
    if (err == cudaSuccess)
      err = gmres_newton(m, w, nb, tol_mismatch, max_newton, gmres_tol, mm, max_outer, precond == 1, st);
    auto o = [&](auto* user, auto* stage, int64_t per) { return dev_ptrs ? (user ? user + s0 * per : nullptr) : (user ? stage : nullptr); };
    if (err == cudaSuccess)
      err = gmres_output(m, w, nb, max_newton, o(theta_out, sth, (int64_t)nbus), o(vmag_out, svm, (int64_t)nbus),
                         o(converged, scv, 1), o(iterations, sit, 1), o(final_mismatch_inf, sfn, 1),
                         o(status, sst, 1), o(gmres_steps, sgs, max_newton), o(gmres_diag, sgd, 1),
                         o(gmres_diag_k, sgk, 1), o(gmres_diag_relres, sdr, 1), st);
    if (!dev_ptrs && err == cudaSuccess) {
      auto back = [&](auto* user, const auto* stage, size_t bytes) {
        if (user && err == cudaSuccess) err = cudaMemcpyAsync(user, stage, bytes, cudaMemcpyDeviceToHost, st);
      };
      back(theta_out + s0 * nbus, sth, nb * nbus * 8);
      back(vmag_out + s0 * nbus, svm, nb * nbus * 8);
      back(converged ? converged + s0 : nullptr, scv, nb);
      back(iterations ? iterations + s0 : nullptr, sit, nb * 4);
      back(final_mismatch_inf ? final_mismatch_inf + s0 : nullptr, sfn, nb * 8);
      back(status ? status + s0 : nullptr, sst, nb * 4);
      back(gmres_steps ? gmres_steps + s0 * max_newton : nullptr, sgs, nb * max_newton * 4);
      back(gmres_diag ? gmres_diag + s0 : nullptr, sgd, nb * 4);
      back(gmres_diag_k ? gmres_diag_k + s0 : nullptr, sgk, nb * 4);
      back(gmres_diag_relres ? gmres_diag_relres + s0 : nullptr, sdr, nb * 8);
    }
    if (err == cudaSuccess) err = cudaStreamSynchronize(st);
  }
  cudaEventRecord(p->ev1, st);
  cudaEventSynchronize(p->ev1);
  float ms = 0.0f;
  cudaEventElapsedTime(&ms, p->ev0, p->ev1);
  p->last_ms = ms;
  ACPF_CUDA(err);
  return ACPF_OK;
}

}  // extern "C"
