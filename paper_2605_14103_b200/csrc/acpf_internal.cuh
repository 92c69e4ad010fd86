// Internal declarations shared by the libacpf translation units.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/acpf.h"

// ACPF_DEBUG_BOUNDS builds (never shipped) turn the index checks at the hot
// gather/scatter sites into device asserts: compute-sanitizer is not
// available on the GPU pool, so bad accesses are caught by our own checks
#ifdef ACPF_DEBUG_BOUNDS
#include <cassert>
#define ACPF_CHECK(cond) assert(cond)
#else
#define ACPF_CHECK(cond) ((void)0)
#endif
#include "nr_symbolic.h"

namespace acpf {

void set_error(const std::string& msg);

constexpr int kGroup = 8;  // NR: scenarios per warp (a quad of lanes each)

// ---------------------------------------------------------------------------
// Newton plan (device side view passed to the kernel by value)
// ---------------------------------------------------------------------------
struct NrDeviceModel {
  int n_bus, n_theta, n_q, n_rows;
  const int32_t* y_rowptr;
  const int32_t* y_col;
  const double2* y_val;
  const double* theta_init;
  const double* vmag_init;
  const int32_t* tpos;     // [n_bus] index into p_spec (theta block) or -1
  const int32_t* qidx;     // [n_bus] index into q_spec (q block) or -1
  const int32_t* bus_row;  // [n_bus] block row of the bus or -1 (slack)
  // level-synchronous 2x2-block Crout schedule (nr_symbolic.h NrSchedule)
  const int32_t* asm_ptr;     // [n_bus+1] Jacobian assembly list per bus
  const double2* asm_y;       // [entries]
  const int32_t* asm_j;       // [entries]
  const int32_t* asm_slot;    // [entries] LU block slot (-1 slack column)
  const uint32_t* slot_info;  // [nnz_lu]
  const int32_t* slot_store;  // [nnz_lu] storage position in the LU region
  const int32_t* row_slot;    // [n_rows+1]
  const int32_t* task_row;    // [n_tasks+1] factor warp tasks (row ranges)
  const int32_t* btask_row;   // [n_btasks+1] back warp tasks (back-order row ranges)
  const int32_t* row_sptr;    // [n_rows+1]
  const uint32_t* brow;       // [n_rows]
  const int32_t* brow_sptr;   // [n_rows+1]
  const uint32_t* stream;     // [n_stream]
  int64_t nnz_lu;
  int64_t n_block, n_scalar;  // arena elements per group (block / scalar region)
  int64_t off_lu, off_yx;                   // block region
  int64_t off_u, off_e, off_spec, off_th, off_vm;     // scalar region
  // LU of the flat-start Jacobian shared by every scenario's first Newton step
  // (nr_flat_start_factor); null when step 0 is factored per scenario
  const double* sh_vals;   // [nnz_lu][4] L^ / inv(D) / U^, row-major 2x2
  const int32_t* sh_col;   // [nnz_lu] block column of the slot
  const int32_t* sh_diag;  // [n_rows] diagonal slot of the row
  const double2* sh_s0;    // [n_bus] S_i at the flat start (step-0 mismatch), or null
  // dense tail (NrSchedule::tail_*): rows tail_row0 .. n_rows-1
  int tail_row0, tail_T, n_tail_slot;
  const int2* tail_slot;   // [n_tail_slot] (storage element, dense block position)
  const int32_t* tail_trow;  // [tail_T] row of each tail-level task, in class order
};

struct NrHostSchedule {
  const int32_t* level_task_ptr;   // [n_levels+1]
  const int32_t* level_maxl;       // [n_levels]
  const int32_t* blevel_task_ptr;  // [n_blevels+1]
  int n_levels, n_blevels, max_l;
  int tail_level;  // factor level of the tail rows (group-major tasks), -1: no tail
  int n_tail_class;
  int tail_variant;  // pipeline shape of the tail level (nr_kernel.cu V0..V3)
  const int32_t* tail_class_ptr;   // [n_tail_class+1] task ranges into tail_trow
  const int32_t* tail_class_maxl;  // [n_tail_class] row-buffer blocks of the class
  int variant;  // factor/back pipeline shape (nr_kernel.cu: 0 = 8x8 ring, 1 = 8x4, 2 = 4x4, 3 = mixed (default))
};

struct NrWorkspace {
  double* arena;  // [groups][block region | scalar region]
  int64_t groups;
  // per scenario [groups*kGroup]
  unsigned long long* fmax_bits;
  int* flags;
  int* status;
  int* iters;
  double* fout;
  uint8_t* active;
  int* gactive;     // [groups]
  int* n_active;    // device counter
  int* host_active; // pinned host mirror
  int* kstep;       // [0] device Newton step counter (kernels read it; graphs stay step-independent),
                    // [1] kernels launched by the device-side loop (nr_count_kernel), summed per solve
};

// Captured per-step launch sequences (CUDA graphs), cached by the plan and
// re-captured when the chunk size, tolerances or workspace change.
struct NrGraphCache {
  cudaStream_t capture = nullptr;  // private stream used only for capture
  cudaGraphExec_t head = nullptr;  // phasor, mismatch, check, D2H of the active count
  cudaGraphExec_t body = nullptr;  // factor levels, back levels, zero-pivot, step++
  cudaGraphExec_t body0 = nullptr; // step 0 with the shared flat-start LU, step++
  int64_t groups = -1, batch = -1;
  double tol = 0.0;
  int max_newton = -1;
  const double* arena = nullptr;
  bool warm = false;  // head/body captured for a warm start (no shared step 0)
  // whole solves with the Newton loop on the device (conditional nodes),
  // one per (chunk size, tolerances, workspace, io pointers) seen recently
  struct Solve {
    cudaGraphExec_t exec = nullptr;
    int64_t batch = -1;
    double tol = 0.0;
    int max_newton = -1;
    const double* arena = nullptr;
    const void* io[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    uint64_t used = 0;
  };
  static constexpr int kSolves = 4;
  Solve solves[kSolves];
  uint64_t tick = 0;
  void release();
};

struct NrBatchIO {
  const double* p_spec;  // [batch][n_theta]
  const double* q_spec;  // [batch][n_q]
  double* theta_out;     // [batch][n_bus]
  double* vmag_out;
  uint8_t* converged;
  int32_t* iterations;
  double* fnorm;
  int32_t* status;
  int64_t batch;  // scenarios in this chunk
  // warm start (acpf_nr_solve_start): [batch][n_bus] start state, or null for
  // the plan's flat start (transmission.py:306-330 `start=`)
  const double* theta_start = nullptr;
  const double* vmag_start = nullptr;
};

// dynamic smem of a factor launch (pipeline variant, longest L part of its rows)
size_t nr_smem_bytes(int variant, int cap);
size_t nr_group_state_bytes();
cudaError_t launch_nr_newton(const NrDeviceModel& m, const NrHostSchedule& hs, const NrWorkspace& w,
                             const NrBatchIO& io, double tol, int max_newton, cudaStream_t stream,
                             int* launches, NrGraphCache* graphs = nullptr);

// ---------------------------------------------------------------------------
// Z-Bus plan
// ---------------------------------------------------------------------------
struct ZbDeviceModel {
  int n;          // non-slack node-phases
  int n_l;        // load columns
  int kpad;       // n_l rounded up to a multiple of 4
  int n_rb;       // row blocks of kZbRows rows
  const double* zfrag;   // fragment-ordered Z[:, l] (see zbus_kernel.cu)
  const double2* v0;     // [n_rb * kZbRows] (zero padded)
  const int32_t* lpos_of_row;  // unused by kernel v1, kept for diagnostics
  const int32_t* l_row;  // [n_l] reduced row of each load column
  const int32_t* wye_l;  // [n_wye] load column of each wye load
  const int32_t* dp_l;   // [n_delta]
  const int32_t* dq_l;   // [n_delta]
  int n_wye, n_delta;
  double floor;
  double mag0;   // sum |v0| with the kernel's own reduction order
};

struct ZbBatchIO {
  const double2* s_wye;   // [batch][n_wye]
  const double2* s_delta; // [batch][n_delta]
  double2* v_out;         // [batch][n]
  uint8_t* converged;
  int32_t* iterations;
  double* final_delta;
  double* residual;
  int32_t* status;
  int32_t* floor_slot;
  int64_t batch;
};

constexpr int kZbRows = 64;  // rows per Z stage

cudaError_t launch_zbus(const ZbDeviceModel& m, const ZbBatchIO& io, double tol, int max_iter,
                        bool mag0_mode, double* mag0_out, int* launches, cudaStream_t stream);
size_t zbus_frag_doubles(int n_rb, int kpad);
void zbus_pack_fragments(const double* zl, int n, int n_l, int n_rb, int kpad, double* out);

// ---------------------------------------------------------------------------
// Seeded scenario generation (scenario_kernel.cu)
// ---------------------------------------------------------------------------
struct NrScenarioArgs {
  uint64_t seed;
  int64_t start, count;
  double spread;
  int n_elem, n_theta, n_q;
  const double* p_base;   // [n_theta] p_gen - p_load over the theta block
  const double* q_base;   // [n_q]
  const int32_t* elem_tpos;
  const int32_t* elem_qidx;
  const double* elem_pl;
  const double* elem_ql;
  const double* elem_pg;
  const double* elem_qg;
  double* p_spec;  // [count][n_theta]
  double* q_spec;  // [count][n_q]
};

struct ZbScenarioArgs {
  uint64_t seed;
  int64_t start, count;
  double spread;
  int n_elem, n_wye, n_delta;
  const int32_t* elem_target;  // >= 0 wye index, else -(delta index)-1
  const double2* wye_s;
  const double2* delta_s;
  double2* s_wye;
  double2* s_delta;
};

cudaError_t launch_philox_multipliers(uint64_t seed, int64_t start, int64_t count, int n_elem,
                                      double spread, double* out, cudaStream_t st);
cudaError_t launch_nr_scenarios(const NrScenarioArgs& a, cudaStream_t st);
cudaError_t launch_zb_scenarios(const ZbScenarioArgs& a, cudaStream_t st);

// ---- certificates (cert_kernel.cu)
struct NrCertModel {
  int n_bus, n_theta, n_q, n_br;
  const int32_t* y_rowptr;
  const int32_t* y_col;
  const double2* y_val;
  const int32_t* tpos;   // [n_bus] p_spec index or -1 (slack)
  const int32_t* qidx;   // [n_bus] q_spec index or -1
  const int32_t* br_f;   // [n_br] from bus
  const int32_t* br_t;   // [n_br] to bus
  const double2* br_y;   // [n_br][4] yff, yft, ytf, ytt
  const double* gs;      // [n_bus] shunt conductance
};

struct NrCertIO {
  int64_t batch;
  const double* theta;   // [batch][n_bus]
  const double* vmag;
  const double* p_spec;  // [batch][n_theta]
  const double* q_spec;  // [batch][n_q]
  double* mismatch_inf;  // [batch] (or null)
  double* slack_balance;
  double* branch_loss;
};

struct ZbCertModel {
  int n, n_wye, n_delta;
  const int32_t* rowptr;  // Y_NN CSR
  const int32_t* col;
  const double2* val;
  const double2* inj;     // [n] Y_NS v_slack
  const int32_t* wye_row;
  const int32_t* dp_row;
  const int32_t* dq_row;
  double floor;
};

struct ZbCertIO {
  int64_t batch;
  const double2* v;        // [batch][n]
  const double2* s_wye;    // [batch][n_wye]
  const double2* s_delta;  // [batch][n_delta]
  double* kcl;             // [batch]
};

acpf_status zbus_reduce_device(int device, int n, const int32_t* rowptr, const int32_t* col, const double* val,
                               const double* rhs0, int n_l, const int32_t* l_index, double* zl_out,
                               double* v0_out, double* min_pivot_out);
void set_error(const std::string& msg);

// ---- GMRES-FD Newton ablation (gmres_kernel.cu)
struct GmModel {
  int n_bus, n_theta, n_q, nj;
  const int32_t* y_rowptr;
  const int32_t* y_col;
  const double2* y_val;
  const int32_t* tpos;
  const int32_t* qidx;
  const int32_t* theta_block;  // [n_theta] bus of each theta unknown
  const int32_t* q_block;      // [n_q]
  const double* theta_init;
  const double* vmag_init;
  const double* binv1;  // [n_theta][n_theta] (B' + eps I)^-1, row-major
  const double* binv2;  // [n_q][n_q]
  const int32_t* g_rowptr;  // G = -Re Y[q, theta] (CSR, n_q rows)
  const int32_t* g_col;
  const double* g_val;
};

struct GmWork {
  int bc;  // scenarios per chunk (vectors are [rows][bc])
  double *th, *vm;
  double2 *u, *ph, *ic, *du;
  double *b, *x, *wv, *t1, *t2, *vb, *h, *cs, *sn, *g, *y, *part;
  double *beta0, *beta, *relres, *scal, *fout;
  const double* p_spec;  // [bc][n_theta] (scenario-major, as the caller's)
  const double* q_spec;
  unsigned long long* fmax_bits;
  int *flags, *nactive, *status, *iters, *gstate, *cyc, *kk, *brk, *gsum, *gtotal, *gdiag, *count;
  int* gsteps;     // [max_newton + 1][bc] GMRES iterations per Newton step
  int* gdiag_k;    // Newton step of the first GMRES diagnostic
  double* gdiag_rel;
  int* host_count;
};

size_t gmres_work_doubles(const GmModel& m, int bc, int restart);
cudaError_t gmres_newton(const GmModel& m, GmWork& w, int64_t nb, double tol, int max_newton,
                         double gtol, int restart, int max_outer, bool fd, cudaStream_t st);
cudaError_t gmres_output(const GmModel& m, const GmWork& w, int64_t nb, int max_newton, double* theta_out,
                         double* vmag_out, uint8_t* converged, int32_t* iterations, double* fnorm,
                         int32_t* status, int32_t* gmres_steps, int32_t* gmres_diag, int32_t* gmres_diag_k,
                         double* gmres_diag_relres, cudaStream_t st);

size_t nr_cert_smem(int n_bus);
size_t zb_cert_smem(int n);
cudaError_t launch_nr_cert(const NrCertModel& m, const NrCertIO& io, cudaStream_t st);
cudaError_t launch_zb_kcl(const ZbCertModel& m, const ZbCertIO& io, cudaStream_t st);

}  // namespace acpf
