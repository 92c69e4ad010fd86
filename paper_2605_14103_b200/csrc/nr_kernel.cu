// Batched polar Newton-Raphson on sm_100a: level-synchronous sparse LU.
//
// Data layout: scenarios are processed in groups of kGroup = 8; each
// scenario owns a quad of lanes (lane = r*8 + sc, sub-lane r = 0..3). Every
// per-scenario quantity lives in a per-group arena of "elements", element e of
// scenario sc at arena[e*8 + sc], so one element of a group is 64 contiguous
// bytes and a warp instruction touching 4 elements moves four fully used
// 64-byte segments. The schedule (Ybus, LU pattern, Crout updates) is shared
// by all groups.
//
// One Newton step of the reference `_newton_loop` (transmission.py:333-380)
// for the whole batch is a short sequence of launches on one stream:
//   nr_phasor    u = V e^{j theta}, E = e^{j theta}; V <= 0 flag  (transmission.py:196, :355)
//   nr_mismatch  I = Y u, S = u conj(I), F -> rhs, ||F||inf, non-finite flags
//                (transmission.py:194-215), and the Jacobian blocks H, N, M, L
//                of every Ybus entry straight into their LU slots
//                (dense_jacobian formulas, transmission.py:383-407)
//   nr_check     the reference exit checks in order: non-finite -> converged
//                -> min V <= 0 -> k == max_newton (transmission.py:347-359)
//   nr_factor    one launch per elimination level: every (row of the level,
//                group) pair is an independent warp task that computes the
//                row by Crout (dot-product) updates + fused forward
//                substitution; rows of one level never read each other
//   nr_back      one launch per back-substitution level
//   nr_update    x += dx (transmission.py:378)
// This replaces the reference's FD-preconditioned GMRES step
// (transmission.py:361-369) by an exact static-pivot sparse LU solve.
//
// Inside a factor/back task every operand that is not produced by the task
// itself (earlier U rows, pivots, y/x, assembled J values) is a precomputed
// element index in a gather stream; the warp runs a cp.async (LDGSTS)
// multistage pipeline over its stream (16 elements per stage, 15 stages =
// 240 elements in flight) into a shared-memory ring, and the quad of a
// scenario splits every dot product 4 ways (partial sums combined by a fixed
// shuffle butterfly). No stream element of a task can be
// produced by another task of the same level, so the pipeline needs no
// hazard checks. The task's own L values stay in shared memory (later rows
// only read U), so global traffic is the U gathers plus one write per U slot.

#include "acpf_internal.cuh"

namespace acpf {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kCh = 16;    // elements per pipeline stage
constexpr int kNBuf = 16;  // stages in the ring (kNBuf-1 in flight)
constexpr int kRing = kCh * kNBuf;
constexpr int kElemBytes = kGroup * 8;  // 64
constexpr int kBusChunk = 64;

__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ double lds_f64(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(a) : "memory");
  return v;
}

__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];\n" : "=r"(v) : "r"(a) : "memory");
  return v;
}

__device__ __forceinline__ void sts_f64(uint32_t a, double v) {
  asm volatile("st.shared.f64 [%0], %1;\n" ::"r"(a), "d"(v) : "memory");
}

__device__ __forceinline__ void sts_u32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;\n" ::"r"(a), "r"(v) : "memory");
}

__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(src) : "memory");
}

__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }

template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// u * conj(a)
__device__ __forceinline__ double2 mul_conj(double2 u, double2 a) {
  return make_double2(u.x * a.x + u.y * a.y, u.y * a.x - u.x * a.y);
}

// sum over the quad of a scenario (lanes sc, sc+8, sc+16, sc+24), fixed order
__device__ __forceinline__ double quad_sum(double x) {
  x = x + __shfl_xor_sync(kFull, x, 8);
  x = x + __shfl_xor_sync(kFull, x, 16);
  return x;
}

// Per-warp gather pipeline over the stream range [s0, s0 + n).
struct Pipe {
  const uint32_t* stream;
  const double* arena;  // group arena base (element e, scenario sc at arena[e*8 + sc])
  uint32_t ring;        // smem [kRing][8] doubles
  uint32_t wring;       // smem [kRing] u32 stream words
  int lane, r, sc;
  int s0, n;            // first stream index, element count
  int issued;           // stages issued
  int ready_upto;       // elements [0, ready_upto) are resident
  int q;                // next element to consume (relative)
  uint32_t wcur, wnext; // word windows: lane j holds the word of element (wbase + j)
  int wbase;

  __device__ __forceinline__ uint32_t load_window(int base) const {
    const int k = base + lane;
    return k < n ? stream[s0 + k] : 0u;
  }

  __device__ __forceinline__ void issue_stage() {
    const int c = issued++;
    const int e0 = c * kCh;
    if (e0 < n) {
      if (e0 >= wbase + 32) {  // advance the double-buffered word window
        wbase += 32;
        wcur = wnext;
        wnext = load_window(wbase + 32);
      }
      const int slot = (c % kNBuf) * kCh;
      const int lim = min(kCh, n - e0);
      const int jw = e0 - wbase;  // 0 or 16
      const uint32_t mine = __shfl_sync(kFull, wcur, (jw + lane) & 31);
      if (lane < lim) sts_u32(wring + (slot + lane) * 4, mine);
#pragma unroll
      for (int j = 0; j < kCh / 4; ++j) {
        const int e = 4 * j + r;
        const uint32_t w = __shfl_sync(kFull, wcur, (jw + e) & 31);
        if (e < lim)
          cp_async8(ring + ((slot + e) * kGroup + sc) * 8, arena + (size_t)(w & 0x3fffffu) * kGroup + sc);
      }
    }
    cp_commit();
  }

  __device__ __forceinline__ void begin(const uint32_t* st, int start, int end) {
    stream = st;
    s0 = start;
    n = end - start;
    issued = 0;
    ready_upto = 0;
    q = 0;
    wbase = 0;
    wcur = load_window(0);
    wnext = load_window(32);
#pragma unroll 1
    for (int k = 0; k < kNBuf - 1; ++k) issue_stage();
  }

  // make element e resident; elements < q must already be consumed
  __device__ __forceinline__ void ensure(int e) {
    while (e >= ready_upto) {
      cp_wait<kNBuf - 2>();
      __syncwarp();
      issue_stage();
      ready_upto += kCh;
    }
  }

  __device__ __forceinline__ uint32_t addr(int e) const {
    return ring + (((e % kRing) * kGroup) + sc) * 8;
  }

  __device__ __forceinline__ uint32_t word(int e) const { return lds_u32(wring + (e % kRing) * 4); }

  // scalar element: every sub-lane reads its scenario's value
  __device__ __forceinline__ double get() {
    ensure(q);
    const double v = lds_f64(addr(q));
    ++q;
    return v;
  }

  __device__ __forceinline__ void finish() {
    cp_wait<0>();
    __syncwarp();
  }
};

#define EL(A, e) (A)[(size_t)(e) * kGroup]

__global__ void nr_init_kernel(NrDeviceModel m, NrWorkspace w, NrBatchIO io) {
  const int lane = threadIdx.x & 31, r = lane >> 3, sc = lane & 7;
  const int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (g >= w.groups) return;
  const int64_t s = g * kGroup + sc;
  const bool valid = s < io.batch;
  double* A = w.arena + (size_t)g * m.n_elem * kGroup + sc;
  for (int i = r; i < m.n_bus; i += 4) {
    EL(A, m.off_th + i) = m.theta_init[i];
    EL(A, m.off_vm + i) = m.vmag_init[i];
  }
  for (int k = r; k < m.n_j; k += 4) {
    double v = 0.0;
    if (valid) v = k < m.n_theta ? io.p_spec[s * m.n_theta + k] : io.q_spec[s * m.n_q + (k - m.n_theta)];
    EL(A, m.off_spec + k) = v;
  }
  if (r) return;
  w.active[s] = valid;
  w.status[s] = 0;
  w.iters[s] = 0;
  w.fout[s] = 0.0;
  w.fmax_bits[s] = 0ull;
  w.flags[s] = 0;
  if (lane == 0) w.gactive[g] = 1;
}

__global__ void nr_phasor_kernel(NrDeviceModel m, NrWorkspace w) {
  const int lane = threadIdx.x & 31, r = lane >> 3, sc = lane & 7;
  const int64_t item = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int nch = (m.n_bus + kBusChunk - 1) / kBusChunk;
  const int64_t g = item / nch;
  if (g >= w.groups || !w.gactive[g]) return;
  const int i0 = (int)(item % nch) * kBusChunk, i1 = min(m.n_bus, i0 + kBusChunk);
  double* A = w.arena + (size_t)g * m.n_elem * kGroup + sc;
  bool neg = false;
  for (int i = i0 + r; i < i1; i += 4) {
    const double t = EL(A, m.off_th + i), v = EL(A, m.off_vm + i);
    double sn, cs;
    sincos(t, &sn, &cs);
    EL(A, m.off_e + 2 * i) = cs;
    EL(A, m.off_e + 2 * i + 1) = sn;
    EL(A, m.off_u + 2 * i) = v * cs;
    EL(A, m.off_u + 2 * i + 1) = v * sn;
    neg |= v <= 0.0;
  }
  if (neg) atomicOr(&w.flags[g * kGroup + sc], 4);
}

__global__ void nr_mismatch_kernel(NrDeviceModel m, NrWorkspace w) {
  const int lane = threadIdx.x & 31, r = lane >> 3, sc = lane & 7;
  const int64_t item = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int nch = (m.n_bus + kBusChunk - 1) / kBusChunk;
  const int64_t g = item / nch;
  if (g >= w.groups || !w.gactive[g]) return;
  const int i0 = (int)(item % nch) * kBusChunk, i1 = min(m.n_bus, i0 + kBusChunk);
  double* A = w.arena + (size_t)g * m.n_elem * kGroup + sc;
  double fmx = 0.0;
  int bad = 0;  // bit0 NaN, bit1 Inf
  for (int i = i0 + r; i < i1; i += 4) {
    double2 acc = make_double2(0.0, 0.0);
    const int e1 = m.y_rowptr[i + 1];
    for (int e = m.y_rowptr[i]; e < e1; ++e) {
      const double2 y = m.y_val[e];
      const int c = m.y_col[e];
      const double ur = EL(A, m.off_u + 2 * c), ui = EL(A, m.off_u + 2 * c + 1);
      acc.x += y.x * ur - y.y * ui;
      acc.y += y.x * ui + y.y * ur;
    }
    const double2 u = make_double2(EL(A, m.off_u + 2 * i), EL(A, m.off_u + 2 * i + 1));
    const double2 sv = mul_conj(u, acc);  // S_i = u_i conj(I_i)
    const int tp = m.tpos[i], qp = m.qpos[i];
    if (tp >= 0) {
      const double f = sv.x - EL(A, m.off_spec + tp);
      bad |= isnan(f) ? 1 : (isinf(f) ? 2 : 0);
      fmx = fmx < fabs(f) ? fabs(f) : fmx;
      EL(A, m.off_yx + m.ipos[tp]) = -f;
    }
    if (qp >= 0) {
      const double f = sv.y - EL(A, m.off_spec + qp);
      bad |= isnan(f) ? 1 : (isinf(f) ? 2 : 0);
      fmx = fmx < fabs(f) ? fabs(f) : fmx;
      EL(A, m.off_yx + m.ipos[qp]) = -f;
    }
    // Jacobian blocks of row bus i into their LU slots:
    //   dS_i/dth_j = -j u_i conj(y u_j)  (j != i);  dS_i/dth_i = j u_i conj(I_i - y u_i)
    //   dS_i/dV_j  =  u_i conj(y E_j) [+ conj(I_i) E_i if j == i]
    //   H = Re dS/dth, N = Re dS/dV, M = Im dS/dth, L = Im dS/dV
    const double2 ei = make_double2(EL(A, m.off_e + 2 * i), EL(A, m.off_e + 2 * i + 1));
    const int a1 = m.asm_ptr[i + 1];
    for (int a = m.asm_ptr[i]; a < a1; ++a) {
      const double2 y = m.asm_y[a];
      const int jb = m.asm_j[a];
      const int4 sl = m.asm_slot[a];
      const double2 ej = make_double2(EL(A, m.off_e + 2 * jb), EL(A, m.off_e + 2 * jb + 1));
      const double2 wv = mul_conj(u, cmul(y, ej));
      double2 dth, dv;
      if (jb != i) {
        const double2 uj = make_double2(EL(A, m.off_u + 2 * jb), EL(A, m.off_u + 2 * jb + 1));
        const double2 wt = mul_conj(u, cmul(y, uj));
        dth = make_double2(wt.y, -wt.x);
        dv = wv;
      } else {
        const double2 yu = cmul(y, u);
        const double2 wt = mul_conj(u, make_double2(acc.x - yu.x, acc.y - yu.y));
        dth = make_double2(-wt.y, wt.x);
        dv = make_double2(wv.x + (acc.x * ei.x + acc.y * ei.y), wv.y + (acc.x * ei.y - acc.y * ei.x));
      }
      if (sl.x >= 0) EL(A, m.off_lu + sl.x) = dth.x;
      if (sl.y >= 0) EL(A, m.off_lu + sl.y) = dv.x;
      if (sl.z >= 0) EL(A, m.off_lu + sl.z) = dth.y;
      if (sl.w >= 0) EL(A, m.off_lu + sl.w) = dv.y;
    }
  }
  const int64_t s = g * kGroup + sc;
  // fmax of non-negative doubles is the max of their bit patterns
  if (fmx > 0.0) atomicMax(&w.fmax_bits[s], (unsigned long long)__double_as_longlong(fmx));
  if (bad) atomicOr(&w.flags[s], bad);
}

__global__ void nr_check_kernel(NrWorkspace w, int64_t batch, int k, int max_newton, double tol) {
  const int lane = threadIdx.x & 31;
  const int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (g >= w.groups) return;
  const int64_t s = g * kGroup + (lane & 7);
  bool act = lane < kGroup && s < batch && w.active[s];
  if (act) {
    const double fmx = __longlong_as_double((long long)w.fmax_bits[s]);
    const int fl = w.flags[s];
    int st = -1;
    double fo = fmx;
    if (fl & 3) {
      st = ACPF_NR_NONFINITE;
      fo = (fl & 1) ? __longlong_as_double(0x7ff8000000000000LL)
                    : __longlong_as_double(0x7ff0000000000000LL);
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
      w.active[s] = 0;
      act = false;
    }
  }
  if (lane < kGroup && s < batch) {
    w.fmax_bits[s] = 0ull;
    w.flags[s] = 0;
  }
  const unsigned any = __ballot_sync(kFull, act);
  if (lane == 0) {
    w.gactive[g] = any != 0;
    if (any) atomicAdd(w.n_active, __popc(any));
  }
}

// One elimination level: task = (row of the level, group).
__global__ void __launch_bounds__(32) nr_factor_kernel(NrDeviceModel m, NrWorkspace w, int r0) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x, r = lane >> 3, sc = lane & 7;
  const int64_t task = blockIdx.x;
  const int64_t g = task % w.groups;
  const int p = r0 + (int)(task / w.groups);
  if (!w.gactive[g]) return;
  double* A = w.arena + (size_t)g * m.n_elem * kGroup + sc;
  const uint32_t ring = su32(smem);
  const uint32_t wring = ring + kRing * kElemBytes;
  const uint32_t lbuf = wring + kRing * 4 + sc * 8;
  Pipe pp;
  pp.arena = w.arena + (size_t)g * m.n_elem * kGroup;
  pp.ring = ring;
  pp.wring = wring;
  pp.lane = lane;
  pp.r = r;
  pp.sc = sc;
  pp.begin(m.stream, m.row_sptr[p], m.row_sptr[p + 1]);
  const int t0 = m.row_slot[p], t1 = m.row_slot[p + 1];
  double yacc = pp.get();  // b_p
  bool zero = false;
  uint32_t winfo = 0;
  for (int t = t0; t < t1; ++t) {
    const int j = (t - t0) & 31;
    if (j == 0) winfo = t + lane < t1 ? m.slot_info[t + lane] : 0u;
    const uint32_t info = __shfl_sync(kFull, winfo, j);
    const int cnt = (int)(info >> 16);
    double a = (info & kSlotFill) ? 0.0 : pp.get();
    if (cnt) {
      // Crout updates split over the quad: sub-lane r takes pairs r, r+4, ...
      double part = 0.0;
      int done = 0;
      while (done < cnt) {
        pp.ensure(pp.q);
        const int nb = min(cnt - done, pp.ready_upto - pp.q);
#pragma unroll 2
        for (int k = r; k < nb; k += 4) {
          const int e = pp.q + k;
          const uint32_t wd = pp.word(e);
          part = fma(-lds_f64(lbuf + (wd >> 22) * kElemBytes), lds_f64(pp.addr(e)), part);
        }
        pp.q += nb;
        done += nb;
      }
      a = a + quad_sum(part);
    }
    if (info & kSlotL) {
      const double inv = pp.get();
      const double yc = pp.get();
      a *= inv;
      yacc = fma(-a, yc, yacc);
      // all quad lanes hold the same value and each writes it, so later
      // reads by a lane depend only on its own store
      sts_f64(lbuf + (t - t0) * kElemBytes, a);
    } else {
      if (info & kSlotDiag) {
        zero |= a == 0.0;
        if (r == 0) EL(A, m.off_invd + p) = 1.0 / a;
      }
      if (r == 0) EL(A, m.off_lu + t) = a;
    }
  }
  if (r == 0) EL(A, m.off_yx + p) = yacc;
  pp.finish();
  if (zero && r == 0) atomicOr(&w.flags[g * kGroup + sc], 8);
}

// One back-substitution level: task = (row of the level, group).
__global__ void __launch_bounds__(32) nr_back_kernel(NrDeviceModel m, NrWorkspace w, int b0) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x, r = lane >> 3, sc = lane & 7;
  const int64_t task = blockIdx.x;
  const int64_t g = task % w.groups;
  const int rr = b0 + (int)(task / w.groups);
  if (!w.gactive[g]) return;
  double* A = w.arena + (size_t)g * m.n_elem * kGroup + sc;
  const uint32_t ring = su32(smem);
  Pipe pp;
  pp.arena = w.arena + (size_t)g * m.n_elem * kGroup;
  pp.ring = ring;
  pp.wring = ring + kRing * kElemBytes;
  pp.lane = lane;
  pp.r = r;
  pp.sc = sc;
  pp.begin(m.stream, m.brow_sptr[rr], m.brow_sptr[rr + 1]);
  const uint32_t b = m.brow[rr];
  const int p = (int)(b & 0xfffffu);
  const int cnt = (int)(b >> 20);
  const double y0 = pp.get();
  const double inv = pp.get();
  double part = 0.0;
  int done = 0;  // (u, x) pairs consumed
  while (done < cnt) {
    pp.ensure(pp.q + 1);  // both elements of the next pair resident
    const int nb = min(cnt - done, (pp.ready_upto - pp.q) >> 1);
    for (int k = r; k < nb; k += 4) {
      const int e = pp.q + 2 * k;
      part = fma(-lds_f64(pp.addr(e)), lds_f64(pp.addr(e + 1)), part);
    }
    pp.q += 2 * nb;
    done += nb;
  }
  const double x = (y0 + quad_sum(part)) * inv;
  if (r == 0) EL(A, m.off_yx + p) = x;
  pp.finish();
}

__global__ void nr_update_kernel(NrDeviceModel m, NrWorkspace w, int k) {
  const int lane = threadIdx.x & 31, r = lane >> 3, sc = lane & 7;
  const int64_t item = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int nch = (m.n_bus + kBusChunk - 1) / kBusChunk;
  const int64_t g = item / nch;
  if (g >= w.groups || !w.gactive[g]) return;
  const int64_t s = g * kGroup + sc;
  if (!w.active[s]) return;
  if (w.flags[s] & 8) {  // zero pivot in this step's factorisation: stop here
    if (item % nch == 0 && r == 0) {
      w.status[s] = ACPF_NR_ZERO_PIVOT;
      w.iters[s] = k;
    }
    return;
  }
  const int i0 = (int)(item % nch) * kBusChunk, i1 = min(m.n_bus, i0 + kBusChunk);
  double* A = w.arena + (size_t)g * m.n_elem * kGroup + sc;
  for (int i = i0 + r; i < i1; i += 4) {
    const int tp = m.tpos[i], qp = m.qpos[i];
    if (tp >= 0) EL(A, m.off_th + i) = EL(A, m.off_th + i) + EL(A, m.off_yx + m.ipos[tp]);
    if (qp >= 0) EL(A, m.off_vm + i) = EL(A, m.off_vm + i) + EL(A, m.off_yx + m.ipos[qp]);
  }
}

// scenarios whose factorisation hit an exact zero pivot stop (state not updated)
__global__ void nr_zero_pivot_kernel(NrWorkspace w, int64_t batch) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= batch || !w.active[s]) return;
  if (w.flags[s] & 8) w.active[s] = 0;
}

__global__ void nr_output_kernel(NrDeviceModel m, NrWorkspace w, NrBatchIO io) {
  const int lane = threadIdx.x & 31, r = lane >> 3, sc = lane & 7;
  const int64_t item = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int nch = (m.n_bus + kBusChunk - 1) / kBusChunk;
  const int64_t g = item / nch;
  if (g >= w.groups) return;
  const int64_t s = g * kGroup + sc;
  if (s >= io.batch) return;
  const int i0 = (int)(item % nch) * kBusChunk, i1 = min(m.n_bus, i0 + kBusChunk);
  const double* A = w.arena + (size_t)g * m.n_elem * kGroup + sc;
  for (int i = i0 + r; i < i1; i += 4) {
    io.theta_out[s * m.n_bus + i] = EL(A, m.off_th + i);
    io.vmag_out[s * m.n_bus + i] = EL(A, m.off_vm + i);
  }
  if (item % nch == 0 && r == 0) {
    const int st = w.status[s];
    if (io.converged) io.converged[s] = st == ACPF_NR_CONVERGED;
    if (io.iterations) io.iterations[s] = w.iters[s];
    if (io.fnorm) io.fnorm[s] = w.fout[s];
    if (io.status) io.status[s] = st;
  }
}

size_t pipe_smem() { return (size_t)kRing * (kElemBytes + 4); }

}  // namespace

size_t nr_smem_bytes(int cap) { return pipe_smem() + (size_t)cap * kElemBytes; }

size_t nr_group_state_bytes() { return kGroup * (8 + 4 + 4 + 4 + 8 + 1) + 4; }

cudaError_t launch_nr_newton(const NrDeviceModel& m, const NrHostSchedule& hs, const NrWorkspace& w,
                             const NrBatchIO& io, double tol, int max_newton, cudaStream_t stream,
                             int* launches) {
  cudaError_t e = cudaFuncSetAttribute(nr_factor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)nr_smem_bytes(hs.max_l));
  if (e != cudaSuccess) return e;
  const int64_t groups = (io.batch + kGroup - 1) / kGroup;
  const int nch = (m.n_bus + kBusChunk - 1) / kBusChunk;
  const int wpb = 4;
  auto blocks = [&](int64_t items) { return (unsigned)((items + wpb - 1) / wpb); };
  int nl = 0;
  nr_init_kernel<<<blocks(groups), 32 * wpb, 0, stream>>>(m, w, io);
  ++nl;
  for (int k = 0; k <= max_newton; ++k) {
    nr_phasor_kernel<<<blocks(groups * nch), 32 * wpb, 0, stream>>>(m, w);
    nr_mismatch_kernel<<<blocks(groups * nch), 32 * wpb, 0, stream>>>(m, w);
    e = cudaMemsetAsync(w.n_active, 0, sizeof(int), stream);
    if (e != cudaSuccess) return e;
    nr_check_kernel<<<blocks(groups), 32 * wpb, 0, stream>>>(w, io.batch, k, max_newton, tol);
    nl += 3;
    e = cudaMemcpyAsync(w.host_active, w.n_active, sizeof(int), cudaMemcpyDeviceToHost, stream);
    if (e != cudaSuccess) return e;
    e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) return e;
    if (*w.host_active == 0) break;
    for (int l = 0; l < hs.n_levels; ++l) {
      const int r0 = hs.level_ptr[l], nr = hs.level_ptr[l + 1] - r0;
      nr_factor_kernel<<<(unsigned)(groups * nr), 32, nr_smem_bytes(hs.level_maxl[l]), stream>>>(m, w, r0);
    }
    for (int l = 0; l < hs.n_blevels; ++l) {
      const int b0 = hs.blevel_ptr[l], nr = hs.blevel_ptr[l + 1] - b0;
      nr_back_kernel<<<(unsigned)(groups * nr), 32, pipe_smem(), stream>>>(m, w, b0);
    }
    nr_update_kernel<<<blocks(groups * nch), 32 * wpb, 0, stream>>>(m, w, k);
    nr_zero_pivot_kernel<<<(unsigned)((io.batch + 255) / 256), 256, 0, stream>>>(w, io.batch);
    nl += hs.n_levels + hs.n_blevels + 2;
  }
  nr_output_kernel<<<blocks(groups * nch), 32 * wpb, 0, stream>>>(m, w, io);
  ++nl;
  if (launches) *launches = nl;
  return cudaGetLastError();
}

}  // namespace acpf
