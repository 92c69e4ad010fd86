// Batched polar Newton-Raphson on sm_100a: level-synchronous 2x2-block sparse LU.
//
// Unknowns are grouped per non-slack bus into 2x2 blocks (theta_i, V_i); a PV
// bus carries a padded V_i with the identity equation dV_i = 0, which leaves
// theta and the PQ magnitudes of the Newton step unchanged. The Jacobian is
// then a block matrix with the Ybus pattern and every stream element, every
// Crout update and every store moves a whole 2x2 block.
//
// Data layout: scenarios are processed in groups of kGroup = 8 and each
// scenario owns a quad of lanes (lane = r*8 + sc): in block operations lane r
// owns entry (r/2, r%2) of every 2x2 block of scenario sc. A per-group arena
// holds a block region (element = 4 entries x 8 scenarios = 256 contiguous
// bytes, entry-major, so one LDGSTS/STG per lane moves a whole element for the
// group) followed by a scalar region (element = 8 scenarios = 64 bytes).
//
// One Newton step of the reference `_newton_loop` (transmission.py:333-380)
// for the whole batch is a short sequence of launches on one stream:
//   nr_phasor    u = V e^{j theta}, E = e^{j theta}; V <= 0 flag  (transmission.py:196, :355)
//   nr_mismatch  I = Y u, S = u conj(I), F -> rhs, ||F||inf, non-finite flags
//                (transmission.py:194-215), and the 2x2 Jacobian block
//                [[H, N], [M, L]] of every Ybus entry straight into its LU slot
//                (dense_jacobian formulas, transmission.py:383-407)
//   nr_check     the reference exit checks in order: non-finite -> converged
//                -> min V <= 0 -> k == max_newton (transmission.py:347-359)
//   nr_factor    one launch per elimination level: every (block row of the
//                level, group) pair is an independent warp task computing the
//                row by block Crout updates + fused forward substitution
//   nr_back      one launch per back-substitution level
//   nr_update    x += dx (transmission.py:378)
// This replaces the reference's FD-preconditioned GMRES step
// (transmission.py:361-369) by an exact sparse LU solve (static 2x2 pivots).
//
// Inside a factor/back task every operand not produced by the task itself
// (earlier U blocks, pivot-block inverses, y/x, assembled J blocks) is a
// precomputed element index in a gather stream; the warp runs a cp.async
// (LDGSTS) multistage pipeline over it (8 elements per stage, 6 stages in
// flight) into a shared-memory ring. No element of a task can be produced by
// another task of the same level, so the pipeline needs no hazard checks.
// The row's own L blocks stay in shared memory (later rows only read U).

#include "acpf_internal.cuh"

namespace acpf {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kCh = 8;     // elements per pipeline stage
constexpr int kNBuf = 8;   // stages in the ring (kNBuf-1 in flight)
constexpr int kRing = kCh * kNBuf;
constexpr int kBlk = 4 * kGroup;      // doubles per block element (32)
constexpr int kBlkBytes = kBlk * 8;   // 256
constexpr int kBusChunk = 64;

__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ double lds_f64(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(a) : "memory");
  return v;
}

__device__ __forceinline__ double2 lds_f64x2(uint32_t a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(a) : "memory");
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

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src) : "memory");
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

// Per-warp gather pipeline over the stream range [s0, s0 + n).
struct Pipe {
  const uint32_t* stream;
  const double* blocks;  // group block region (element e at blocks + e*32)
  uint32_t ring;         // smem [kRing] elements of 256 B
  uint32_t wring;        // smem [kRing] u32 stream words
  int lane;
  int s0, n, issued, ready_upto, q;
  uint32_t wcur, wnext;  // word windows: lane j holds the word of element (wbase + j)
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
      const int jw = e0 - wbase;
      const uint32_t mine = __shfl_sync(kFull, wcur, (jw + lane) & 31);
      if (lane < lim) sts_u32(wring + (slot + lane) * 4, mine);
      // 16 B per lane: lanes 0-15 copy element j, lanes 16-31 element j+1
      const int half = lane >> 4, chunk = lane & 15;
#pragma unroll
      for (int j = 0; j < kCh; j += 2) {
        const int jj = j + half;
        const uint32_t w = __shfl_sync(kFull, wcur, (jw + jj) & 31);
        if (jj < lim)
          cp_async16(ring + (slot + jj) * kBlkBytes + chunk * 16,
                     blocks + (size_t)(w & 0x3fffffu) * kBlk + chunk * 2);
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
    for (int k = 0; k < kNBuf - 2; ++k) issue_stage();
  }

  // Make element e resident. Callers keep e <= q + 1 (q = first element not
  // yet consumed). kNBuf-2 stages are in flight, so the stage issued here
  // reuses the slot of stage (e/kCh - 2), which is fully consumed.
  __device__ __forceinline__ void ensure(int e) {
    while (e >= ready_upto) {
      cp_wait<kNBuf - 3>();
      __syncwarp();
      issue_stage();
      ready_upto += kCh;
    }
  }

  // smem address of entry `ent` (0..3) of element e for scenario sc
  __device__ __forceinline__ uint32_t addr(int e, int ent, int sc) const {
    return ring + (e % kRing) * kBlkBytes + (sc * 4 + ent) * 8;
  }

  __device__ __forceinline__ uint32_t word(int e) const { return lds_u32(wring + (e % kRing) * 4); }

  __device__ __forceinline__ uint32_t slot_base(int e) const { return ring + (e % kRing) * kBlkBytes; }

  __device__ __forceinline__ void finish() {
    cp_wait<0>();
    __syncwarp();
  }
};

// block-region entry `ent` of block element e, scenario sc (B = group block base + 4*sc).
// Elements are scenario-major (4 consecutive entries per scenario). Matrix
// blocks are stored column-major: entry (i, j) at 2*j + i.
#define BL(B, e, ent) (B)[(size_t)(e) * kBlk + (ent)]
// scalar-region element e, scenario sc (S = group scalar base + sc)
#define SL(S, e) (S)[(size_t)(e) * kGroup]

struct GroupBase {
  double* b;  // block region + sc
  double* s;  // scalar region + sc
};

__device__ __forceinline__ GroupBase group_base(const NrDeviceModel& m, const NrWorkspace& w, int64_t g,
                                                int sc) {
  double* base = w.arena + (size_t)g * (m.n_block * kBlk + m.n_scalar * kGroup);
  return GroupBase{base + 4 * sc, base + m.n_block * kBlk + sc};
}

__global__ void nr_init_kernel(NrDeviceModel m, NrWorkspace w, NrBatchIO io) {
  const int lane = threadIdx.x & 31, r = lane >> 3, sc = lane & 7;
  const int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (g >= w.groups) return;
  const int64_t s = g * kGroup + sc;
  const bool valid = s < io.batch;
  const GroupBase gb = group_base(m, w, g, sc);
  for (int i = r; i < m.n_bus; i += 4) {
    SL(gb.s, m.off_th + i) = m.theta_init[i];
    SL(gb.s, m.off_vm + i) = m.vmag_init[i];
    const int p = m.bus_row[i];
    if (p >= 0) {
      const int tp = m.tpos[i], qi = m.qidx[i];
      SL(gb.s, m.off_spec + 2 * p) = valid ? io.p_spec[s * m.n_theta + tp] : 0.0;
      SL(gb.s, m.off_spec + 2 * p + 1) = (valid && qi >= 0) ? io.q_spec[s * m.n_q + qi] : 0.0;
    }
  }
  if (r) return;
  w.active[s] = valid;
  w.status[s] = 0;
  w.iters[s] = 0;
  w.fout[s] = 0.0;
  w.fmax_bits[s] = 0ull;
  w.flags[s] = 0;
  if (sc == 0) w.gactive[g] = 1;
}

__global__ void nr_phasor_kernel(NrDeviceModel m, NrWorkspace w) {
  const int lane = threadIdx.x & 31, r = lane >> 3, sc = lane & 7;
  const int64_t item = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int nch = (m.n_bus + kBusChunk - 1) / kBusChunk;
  const int64_t g = item / nch;
  if (g >= w.groups || !w.gactive[g]) return;
  const int i0 = (int)(item % nch) * kBusChunk, i1 = min(m.n_bus, i0 + kBusChunk);
  const GroupBase gb = group_base(m, w, g, sc);
  bool neg = false;
  for (int i = i0 + r; i < i1; i += 4) {
    const double t = SL(gb.s, m.off_th + i), v = SL(gb.s, m.off_vm + i);
    double sn, cs;
    sincos(t, &sn, &cs);
    SL(gb.s, m.off_e + 2 * i) = cs;
    SL(gb.s, m.off_e + 2 * i + 1) = sn;
    SL(gb.s, m.off_u + 2 * i) = v * cs;
    SL(gb.s, m.off_u + 2 * i + 1) = v * sn;
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
  const GroupBase gb = group_base(m, w, g, sc);
  double fmx = 0.0;
  int bad = 0;  // bit0 NaN, bit1 Inf
  for (int i = i0 + r; i < i1; i += 4) {
    const int p = m.bus_row[i];
    if (p < 0) continue;  // slack: no equations
    double2 acc = make_double2(0.0, 0.0);
    const int e1 = m.y_rowptr[i + 1];
    for (int e = m.y_rowptr[i]; e < e1; ++e) {
      const double2 y = m.y_val[e];
      const int c = m.y_col[e];
      const double ur = SL(gb.s, m.off_u + 2 * c), ui = SL(gb.s, m.off_u + 2 * c + 1);
      acc.x += y.x * ur - y.y * ui;
      acc.y += y.x * ui + y.y * ur;
    }
    const double2 u = make_double2(SL(gb.s, m.off_u + 2 * i), SL(gb.s, m.off_u + 2 * i + 1));
    const double2 sv = mul_conj(u, acc);  // S_i = u_i conj(I_i)
    const bool pq = m.qidx[i] >= 0;
    const double fp = sv.x - SL(gb.s, m.off_spec + 2 * p);
    bad |= isnan(fp) ? 1 : (isinf(fp) ? 2 : 0);
    fmx = fmx < fabs(fp) ? fabs(fp) : fmx;
    BL(gb.b, m.off_yx + p, 0) = -fp;
    double fq = 0.0;
    if (pq) {
      fq = sv.y - SL(gb.s, m.off_spec + 2 * p + 1);
      bad |= isnan(fq) ? 1 : (isinf(fq) ? 2 : 0);
      fmx = fmx < fabs(fq) ? fabs(fq) : fmx;
    }
    BL(gb.b, m.off_yx + p, 1) = -fq;
    // 2x2 Jacobian block of every Ybus entry (i, j) into its LU slot:
    //   dS_i/dth_j = -j u_i conj(y u_j)  (j != i);  dS_i/dth_i = j u_i conj(I_i - y u_i)
    //   dS_i/dV_j  =  u_i conj(y E_j) [+ conj(I_i) E_i if j == i]
    //   [[H, N], [M, L]] = [[Re dS/dth, Re dS/dV], [Im dS/dth, Im dS/dV]]
    // with the PV padding rows/columns of the identity equation dV = 0.
    const double2 ei = make_double2(SL(gb.s, m.off_e + 2 * i), SL(gb.s, m.off_e + 2 * i + 1));
    const int a1 = m.asm_ptr[i + 1];
    for (int a = m.asm_ptr[i]; a < a1; ++a) {
      const int slot = m.asm_slot[a];
      if (slot < 0) continue;  // slack column
      const double2 y = m.asm_y[a];
      const int jb = m.asm_j[a];
      const double2 ej = make_double2(SL(gb.s, m.off_e + 2 * jb), SL(gb.s, m.off_e + 2 * jb + 1));
      const double2 wv = mul_conj(u, cmul(y, ej));
      double2 dth, dv;
      if (jb != i) {
        const double2 uj = make_double2(SL(gb.s, m.off_u + 2 * jb), SL(gb.s, m.off_u + 2 * jb + 1));
        const double2 wt = mul_conj(u, cmul(y, uj));
        dth = make_double2(wt.y, -wt.x);
        dv = wv;
      } else {
        const double2 yu = cmul(y, u);
        const double2 wt = mul_conj(u, make_double2(acc.x - yu.x, acc.y - yu.y));
        dth = make_double2(-wt.y, wt.x);
        dv = make_double2(wv.x + (acc.x * ei.x + acc.y * ei.y), wv.y + (acc.x * ei.y - acc.y * ei.x));
      }
      const bool pqj = m.qidx[jb] >= 0;
      // column-major [[H, N], [M, L]]: H (0,0)->0, M (1,0)->1, N (0,1)->2, L (1,1)->3
      BL(gb.b, m.off_lu + slot, 0) = dth.x;
      BL(gb.b, m.off_lu + slot, 1) = pq ? dth.y : 0.0;
      BL(gb.b, m.off_lu + slot, 2) = pqj ? dv.x : 0.0;
      BL(gb.b, m.off_lu + slot, 3) = (pq && pqj) ? dv.y : (jb == i ? 1.0 : 0.0);
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

// One elimination level: task = (run of block rows of the level, group).
// Lane (r, sc) owns entry (i, j) = (r/2, r%2) of every block of scenario sc.
__global__ void __launch_bounds__(32) nr_factor_kernel(NrDeviceModel m, NrWorkspace w, int task0) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x, r = lane >> 3, sc = lane & 7;
  const int bi = r >> 1, bj = r & 1;
  const int64_t task = blockIdx.x;
  const int64_t g = task % w.groups;
  const int tk = task0 + (int)(task / w.groups);
  if (!w.gactive[g]) return;
  const GroupBase gb = group_base(m, w, g, sc);
  const uint32_t ring = su32(smem);
  const uint32_t wring = ring + kRing * kBlkBytes;
  const uint32_t lbuf = wring + kRing * 4;
  // lbuf holds the row's L blocks row-major: entry (i, j) of scenario sc at
  // lbuf + pos*256 + (4*sc + 2*i + j)*8, so L[i][0..1] is one 16-byte load;
  // U blocks are column-major so U[0..1][j] is one 16-byte load too
  const uint32_t offL = (4 * sc + 2 * bi) * 8;   // L[i][0], L[i][1]
  const uint32_t offU = (4 * sc + 2 * bj) * 8;   // U[0][j], U[1][j] (column j)
  const int ce = 2 * bj + bi;                     // this lane's column-major entry
  const int p0 = m.task_row[tk], p1 = m.task_row[tk + 1];
  Pipe pp;
  pp.blocks = w.arena + (size_t)g * (m.n_block * kBlk + m.n_scalar * kGroup);
  pp.ring = ring;
  pp.wring = wring;
  pp.lane = lane;
  pp.begin(m.stream, m.row_sptr[p0], m.row_sptr[p1]);
  bool zero = false;
  // slot control words of the whole task (lane j holds slot tw + j), double
  // buffered so the next window's load is in flight a window ahead
  const int ts0 = m.row_slot[p0], ts1 = m.row_slot[p1];
  int tw = ts0;
  uint32_t winfo = ts0 + lane < ts1 ? m.slot_info[ts0 + lane] : 0u;
  uint32_t ninfo = ts0 + 32 + lane < ts1 ? m.slot_info[ts0 + 32 + lane] : 0u;
  int t = ts0;
  for (int p = p0; p < p1; ++p) {
    const int t0 = t;
    pp.ensure(pp.q);
    double yacc = lds_f64(pp.addr(pp.q, bi, sc));  // b_p[i]
    ++pp.q;
    for (;; ++t) {
      if (t - tw == 32) {
        tw += 32;
        winfo = ninfo;
        ninfo = tw + 32 + lane < ts1 ? m.slot_info[tw + 32 + lane] : 0u;
      }
      const uint32_t info = __shfl_sync(kFull, winfo, t - tw);
      const int cnt = (int)(info >> 16);
      double a = 0.0, a2 = 0.0;
      if (!(info & kSlotFill)) {
        pp.ensure(pp.q);
        a = lds_f64(pp.addr(pp.q, ce, sc));
        ++pp.q;
      }
      // block Crout updates: A_pt -= L_pm U_mt, lane owns (i, j); two
      // interleaved accumulator pairs keep four independent FMA chains
      double a3 = 0.0, a4 = 0.0;
      for (int q = 0; q < cnt;) {
        pp.ensure(pp.q);
        const int nb = min(cnt - q, pp.ready_upto - pp.q);
        int k = 0;
        for (; k + 1 < nb; k += 2) {
          const int e = pp.q + k;
          const uint32_t w0 = pp.word(e), w1 = pp.word(e + 1);
          const double2 l0 = lds_f64x2(lbuf + (w0 >> 22) * kBlkBytes + offL);
          const double2 l1 = lds_f64x2(lbuf + (w1 >> 22) * kBlkBytes + offL);
          const double2 u0 = lds_f64x2(pp.slot_base(e) + offU);
          const double2 u1 = lds_f64x2(pp.slot_base(e + 1) + offU);
          a = fma(-l0.x, u0.x, a);
          a2 = fma(-l0.y, u0.y, a2);
          a3 = fma(-l1.x, u1.x, a3);
          a4 = fma(-l1.y, u1.y, a4);
        }
        if (k < nb) {
          const int e = pp.q + k;
          const double2 l0 = lds_f64x2(lbuf + (pp.word(e) >> 22) * kBlkBytes + offL);
          const double2 u0 = lds_f64x2(pp.slot_base(e) + offU);
          a = fma(-l0.x, u0.x, a);
          a2 = fma(-l0.y, u0.y, a2);
        }
        pp.q += nb;
        q += nb;
      }
      a = (a + a3) + (a2 + a4);
      if (info & kSlotL) {
        pp.ensure(pp.q + 1);
        const int e = pp.q;
        // L_pt = A' inv(U_tt); y_p -= L_pt y_t
        const double o = __shfl_xor_sync(kFull, a, 8);  // entry (i, 1-j)
        const double ai0 = bj ? o : a, ai1 = bj ? a : o;
        const double2 iv = lds_f64x2(pp.slot_base(e) + offU);  // inv[0][j], inv[1][j]
        const double l = ai0 * iv.x + ai1 * iv.y;
        sts_f64(lbuf + (t - t0) * kBlkBytes + (4 * sc + 2 * bi + bj) * 8, l);
        const double lo = __shfl_xor_sync(kFull, l, 8);
        const double li0 = bj ? lo : l, li1 = bj ? l : lo;
        const double2 yt = lds_f64x2(pp.slot_base(e + 1) + 4 * sc * 8);
        yacc = fma(-li1, yt.y, fma(-li0, yt.x, yacc));
        pp.q += 2;
      } else {
        if (info & kSlotDiag) {
          const double a00 = __shfl_sync(kFull, a, sc), a01 = __shfl_sync(kFull, a, 8 + sc);
          const double a10 = __shfl_sync(kFull, a, 16 + sc), a11 = __shfl_sync(kFull, a, 24 + sc);
          const double det = a00 * a11 - a01 * a10;
          zero |= det == 0.0;
          const double rd = 1.0 / det;
          const double inv = r == 0 ? a11 * rd : (r == 1 ? -a01 * rd : (r == 2 ? -a10 * rd : a00 * rd));
          BL(gb.b, m.off_invd + p, ce) = inv;
        }
        BL(gb.b, m.off_lu + t, ce) = a;
      }
      if (info & kSlotRowEnd) {
        ++t;
        break;
      }
    }
    if (bj == 0) BL(gb.b, m.off_yx + p, bi) = yacc;
    __syncwarp();  // lbuf of this row complete before the next row of the task reuses it
  }
  pp.finish();
  if (zero && r == 0) atomicOr(&w.flags[g * kGroup + sc], 8);
}

// One back-substitution level: task = (run of back rows of the level, group).
__global__ void __launch_bounds__(32) nr_back_kernel(NrDeviceModel m, NrWorkspace w, int task0) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x, r = lane >> 3, sc = lane & 7;
  const int bi = r >> 1, bj = r & 1;
  const int64_t task = blockIdx.x;
  const int64_t g = task % w.groups;
  const int tk = task0 + (int)(task / w.groups);
  if (!w.gactive[g]) return;
  const GroupBase gb = group_base(m, w, g, sc);
  const uint32_t ring = su32(smem);
  const int r0 = m.btask_row[tk], r1 = m.btask_row[tk + 1];
  Pipe pp;
  pp.blocks = w.arena + (size_t)g * (m.n_block * kBlk + m.n_scalar * kGroup);
  pp.ring = ring;
  pp.wring = ring + kRing * kBlkBytes;
  pp.lane = lane;
  pp.begin(m.stream, m.brow_sptr[r0], m.brow_sptr[r1]);
  // back-row words of the task (lane j holds row rw + j), double buffered
  int rw = r0;
  uint32_t wrow = r0 + lane < r1 ? m.brow[r0 + lane] : 0u;
  uint32_t nrow = r0 + 32 + lane < r1 ? m.brow[r0 + 32 + lane] : 0u;
  for (int rr = r0; rr < r1; ++rr) {
    if (rr - rw == 32) {
      rw += 32;
      wrow = nrow;
      nrow = rw + 32 + lane < r1 ? m.brow[rw + 32 + lane] : 0u;
    }
    const uint32_t b = __shfl_sync(kFull, wrow, rr - rw);
    const int p = (int)(b & 0xfffffu);
    const int cnt = (int)(b >> 20);
    pp.ensure(pp.q + 1);
    const double yi = lds_f64(pp.addr(pp.q, bi, sc));
    const double inv0 = lds_f64(pp.addr(pp.q + 1, bi, sc));
    const double inv1 = lds_f64(pp.addr(pp.q + 1, 2 + bi, sc));
    pp.q += 2;
    double part = 0.0;  // sum_c U_pc[i][j] x_c[j]
    for (int q = 0; q < cnt;) {
      pp.ensure(pp.q + 1);
      const int nb = min(cnt - q, (pp.ready_upto - pp.q) >> 1);
      for (int k = 0; k < nb; ++k) {
        const int e = pp.q + 2 * k;
        part = fma(lds_f64(pp.addr(e, 2 * bj + bi, sc)), lds_f64(pp.addr(e + 1, bj, sc)), part);
      }
      pp.q += 2 * nb;
      q += nb;
    }
    const double po = __shfl_xor_sync(kFull, part, 8);
    const double acc = yi - (bj ? po + part : part + po);  // (y_p - sum)[i]
    const double ao = __shfl_xor_sync(kFull, acc, 16);     // the other row
    const double acc0 = bi ? ao : acc, acc1 = bi ? acc : ao;
    const double x = inv0 * acc0 + inv1 * acc1;            // x_p[i]
    if (bj == 0) BL(gb.b, m.off_yx + p, bi) = x;
  }
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
  const GroupBase gb = group_base(m, w, g, sc);
  for (int i = i0 + r; i < i1; i += 4) {
    const int p = m.bus_row[i];
    if (p < 0) continue;
    SL(gb.s, m.off_th + i) = SL(gb.s, m.off_th + i) + BL(gb.b, m.off_yx + p, 0);
    if (m.qidx[i] >= 0) SL(gb.s, m.off_vm + i) = SL(gb.s, m.off_vm + i) + BL(gb.b, m.off_yx + p, 1);
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
  const GroupBase gb = group_base(m, w, g, sc);
  for (int i = i0 + r; i < i1; i += 4) {
    io.theta_out[s * m.n_bus + i] = SL(gb.s, m.off_th + i);
    io.vmag_out[s * m.n_bus + i] = SL(gb.s, m.off_vm + i);
  }
  if (item % nch == 0 && r == 0) {
    const int st = w.status[s];
    if (io.converged) io.converged[s] = st == ACPF_NR_CONVERGED;
    if (io.iterations) io.iterations[s] = w.iters[s];
    if (io.fnorm) io.fnorm[s] = w.fout[s];
    if (io.status) io.status[s] = st;
  }
}

size_t pipe_smem() { return (size_t)kRing * (kBlkBytes + 4); }

}  // namespace

size_t nr_smem_bytes(int cap) { return pipe_smem() + (size_t)cap * kBlkBytes; }

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
      const int k0 = hs.level_task_ptr[l], nt = hs.level_task_ptr[l + 1] - k0;
      nr_factor_kernel<<<(unsigned)(groups * nt), 32, nr_smem_bytes(hs.level_maxl[l]), stream>>>(m, w, k0);
    }
    for (int l = 0; l < hs.n_blevels; ++l) {
      const int k0 = hs.blevel_task_ptr[l], nt = hs.blevel_task_ptr[l + 1] - k0;
      nr_back_kernel<<<(unsigned)(groups * nt), 32, pipe_smem(), stream>>>(m, w, k0);
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
