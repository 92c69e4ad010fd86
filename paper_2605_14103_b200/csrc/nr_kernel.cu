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
// bytes, two block-column halves of 128 B; see BL) followed by a scalar region
// (element = 8 scenarios = 64 bytes).
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
//                row by block Crout updates + fused forward substitution, in
//                the unit-upper form A = L^ U^ (L^ = L D, U^ = D^-1 U with
//                D = diag(U_pp)): the pivot inverse stays in registers for the
//                row's own U^ blocks and y_p, so no later row or the back
//                substitution ever gathers a pivot inverse
//   nr_back      one launch per back-substitution level
//   (next step) nr_phasor applies x += dx (transmission.py:378) first
// This replaces the reference's FD-preconditioned GMRES step
// (transmission.py:361-369) by an exact sparse LU solve (static 2x2 pivots).
//
// Inside a factor/back task every operand not produced by the task itself
// (earlier U^ blocks, y/x, assembled J blocks) is a
// precomputed element index in a gather stream; the warp runs a cp.async
// (LDGSTS) multistage pipeline over it into a small shared-memory ring
// (PipeLdgsts; 4- or 8-element stages, 2 stages in flight, so ~20 warps stay
// resident per SM). No element of a task can be produced by another task of
// the same level, so the pipeline needs no hazard checks. The row's own L
// blocks stay in shared memory (later rows only read U).

#include "acpf_internal.cuh"

#include <cstdlib>

namespace acpf {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kBlk = 4 * kGroup;      // doubles per block element (32)
constexpr int kBlkBytes = kBlk * 8;   // 256
constexpr int kHalf = kBlkBytes / 2;  // bytes of one block column of the group (128)
#ifndef ACPF_NR_BUS_CHUNK
#define ACPF_NR_BUS_CHUNK 16  // 64: mismatch 9.6 ms, 16: 8.3 ms, 8: 8.0 ms, 4: 10.7 ms (gb2224 x 65536)
#endif
constexpr int kBusChunk = ACPF_NR_BUS_CHUNK;  // buses per warp in the per-bus kernels

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

// Per-warp gather pipeline over the stream range [s0, s0 + n) for a unit of
// NG consecutive scenario groups. A ring slot holds one stream element of all
// NG groups (NG x 256 B, group h at +256h); CH elements per stage, NBUF
// stages in the ring.
template <int NG_, int CH_, int NBUF_>
struct PipeLdgsts {
  static constexpr int NG = NG_, CH = CH_, NBUF = NBUF_;
  static constexpr int kSlot = NG * kBlkBytes;
  static constexpr int kRingN = CH * NBUF;
  static_assert((kRingN & (kRingN - 1)) == 0, "ring size must be a power of two");
  const uint32_t* stream;
  const double* src;  // this lane's copy source: its group's block region + chunk
  uint32_t n_elem;    // block elements per group (bounds checks)
  bool cp_ok;         // this lane's group is live (NG = 2: lanes 16-31 copy group 1)
  int nlive;          // live groups of the unit
  uint32_t ring;      // smem [kRingN] slots
  uint32_t wring;     // smem [kRingN] u32 stream words
  int lane;
  int s0, n, issued, ready_upto, q;
  uint32_t wcur, wnext;  // word windows: lane j holds the word of element (wbase + j)
  int wbase;

  static constexpr size_t kSmem = (size_t)kRingN * (kSlot + 4);
  __host__ __device__ static constexpr size_t smem_bytes() { return kSmem; }

  __device__ __forceinline__ uint32_t load_window(int base) const {
    const int k = base + lane;
    return k < n ? stream[s0 + k] : 0u;
  }

  __device__ __forceinline__ void issue_stage() {
    const int c = issued++;
    const int e0 = c * CH;
    if (e0 < n) {
      if (e0 >= wbase + 32) {  // advance the double-buffered word window
        wbase += 32;
        wcur = wnext;
        wnext = load_window(wbase + 32);
      }
      const int slot = (c % NBUF) * CH;
      const int lim = min(CH, n - e0);
      const int jw = e0 - wbase;
      // the consumer only needs the L position, pre-scaled to a byte offset
      const uint32_t mine = __shfl_sync(kFull, wcur, (jw + lane) & 31);
      if (lane < lim) sts_u32(wring + (slot + lane) * 4, (mine >> 22) * (uint32_t)kSlot);
      if (NG == 1) {
        // 16 B per lane: lanes 0-15 copy element j, lanes 16-31 element j+1
        const int half = lane >> 4, chunk = lane & 15;
#pragma unroll
        for (int j = 0; j < CH; j += 2) {
          const int jj = j + half;
          const uint32_t w = __shfl_sync(kFull, wcur, (jw + jj) & 31);
          ACPF_CHECK(jj >= lim || (w & 0x3fffffu) < n_elem);
          if (jj < lim) cp_async16(ring + (slot + jj) * kSlot + chunk * 16, src + (size_t)(w & 0x3fffffu) * kBlk);
        }
      } else {
        // one element per instruction: lanes 0-15 group 0, lanes 16-31 group 1
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          const uint32_t w = __shfl_sync(kFull, wcur, (jw + j) & 31);
          ACPF_CHECK(j >= lim || (w & 0x3fffffu) < n_elem);
          if (j < lim && cp_ok) cp_async16(ring + (slot + j) * kSlot + lane * 16, src + (size_t)(w & 0x3fffffu) * kBlk);
        }
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
    for (int k = 0; k < NBUF - 2; ++k) issue_stage();
  }

  // Make element e resident. Callers keep e <= q + 1 (q = first element not
  // yet consumed). NBUF-2 stages are in flight, so the stage issued here
  // reuses the slot of stage (e/CH - 2), which is fully consumed.
  __device__ __forceinline__ void ensure(int e) {
    while (e >= ready_upto) {
      cp_wait<NBUF - 3>();
      __syncwarp();
      issue_stage();
      ready_upto += CH;
    }
  }

  __device__ __forceinline__ uint32_t slot_base(int e) const {
    return ring + ((uint32_t)e % (uint32_t)kRingN) * kSlot;
  }

  // byte offset of element e's L block in the row buffer (lpos * kSlot)
  __device__ __forceinline__ uint32_t lofs(int e) const {
    return lds_u32(wring + ((uint32_t)e % (uint32_t)kRingN) * 4);
  }

  __device__ __forceinline__ void finish() {
    cp_wait<0>();
    __syncwarp();
  }
};

// block-region entry `ent` of block element e, scenario sc (B = group block base + 2*sc).
// An element is two 128-byte column halves: entry (i, j) of scenario sc at
// double 16*j + 2*sc + i, so the 8 lanes of a quarter-warp that read column j
// (or a row-major L row i) of their 8 scenarios touch one contiguous 128 B
// (conflict-free 16-byte shared loads).
#define BL(B, e, ent) (B)[(size_t)(e) * kBlk + ((ent) >> 1) * (2 * kGroup) + ((ent) & 1)]
// scalar-region element e, scenario sc (S = group scalar base + sc)
#define SL(S, e) (S)[(size_t)(e) * kGroup]

struct GroupBase {
  double* b;  // block region + sc
  double* s;  // scalar region + sc
};

__device__ __forceinline__ GroupBase group_base(const NrDeviceModel& m, const NrWorkspace& w, int64_t g,
                                                int sc) {
  double* base = w.arena + (size_t)g * (m.n_block * kBlk + m.n_scalar * kGroup);
  return GroupBase{base + 2 * sc, base + m.n_block * kBlk + sc};
}

__global__ void nr_init_kernel(NrDeviceModel m, NrWorkspace w, NrBatchIO io) {
  const int lane = threadIdx.x & 31, r = lane >> 3, sc = lane & 7;
  const int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (g >= w.groups) return;
  const int64_t s = g * kGroup + sc;
  const bool valid = s < io.batch;
  const GroupBase gb = group_base(m, w, g, sc);
  const bool warm = io.theta_start != nullptr && valid;
  for (int i = r; i < m.n_bus; i += 4) {
    SL(gb.s, m.off_th + i) = warm ? io.theta_start[s * m.n_bus + i] : m.theta_init[i];
    SL(gb.s, m.off_vm + i) = warm ? io.vmag_start[s * m.n_bus + i] : m.vmag_init[i];
    const int p = m.bus_row[i];
    if (p >= 0) {
      const int tp = m.tpos[i], qi = m.qidx[i];
      SL(gb.s, m.off_spec + 2 * p) = valid ? io.p_spec[s * m.n_theta + tp] : 0.0;
      SL(gb.s, m.off_spec + 2 * p + 1) = (valid && qi >= 0) ? io.q_spec[s * m.n_q + qi] : 0.0;
    }
  }
  if (r) return;
  if (g == 0 && sc == 0) *w.kstep = 0;
  w.active[s] = valid;
  w.status[s] = 0;
  w.iters[s] = 0;
  w.fout[s] = 0.0;
  w.fmax_bits[s] = 0ull;
  w.flags[s] = 0;
  if (sc == 0) w.gactive[g] = 1;
}

// Applies the previous step's correction x += dx (transmission.py:378) to the
// scenarios still active (`apply`, every step but the first; scenarios whose
// factorisation hit a zero pivot were deactivated by nr_zero_pivot_kernel),
// then u = V e^{j theta}, E = e^{j theta} and the V <= 0 flag.
__global__ void nr_phasor_kernel(NrDeviceModel m, NrWorkspace w) {
  const int lane = threadIdx.x & 31, r = lane >> 3, sc = lane & 7;
  const int64_t item = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (item == 0 && threadIdx.x == 0) *w.n_active = 0;  // nr_check_kernel counts into it after this launch
  const int nch = (m.n_bus + kBusChunk - 1) / kBusChunk;
  const int64_t g = item / nch;
  if (g >= w.groups || !w.gactive[g]) return;
  const int i0 = (int)(item % nch) * kBusChunk, i1 = min(m.n_bus, i0 + kBusChunk);
  const GroupBase gb = group_base(m, w, g, sc);
  const int k = *w.kstep;
  const bool upd = k > 0 && w.active[g * kGroup + sc];
  bool neg = false;
  if (k == 0 && m.sh_s0) return;  // flat start: S_i shared (nr_mismatch_kernel), V > 0 checked on the host
  // one bus: loads (state, correction) separated from the update so that two
  // buses' loads are in flight together (same arithmetic)
  struct Bus {
    double t, v, dt, dv;
    int p;
    bool q;
  };
  auto load = [&](int i) {
    Bus b{SL(gb.s, m.off_th + i), SL(gb.s, m.off_vm + i), 0.0, 0.0, -1, false};
    if (upd) {
      b.p = m.bus_row[i];
      if (b.p >= 0) {
        b.q = m.qidx[i] >= 0;
        b.dt = BL(gb.b, m.off_yx + b.p, 0);
        if (b.q) b.dv = BL(gb.b, m.off_yx + b.p, 1);
      }
    }
    return b;
  };
  auto finish = [&](int i, Bus b) {
    if (b.p >= 0) {
      b.t = b.t + b.dt;
      SL(gb.s, m.off_th + i) = b.t;
      if (b.q) {
        b.v = b.v + b.dv;
        SL(gb.s, m.off_vm + i) = b.v;
      }
    }
    double sn, cs;
    sincos(b.t, &sn, &cs);
    SL(gb.s, m.off_u + 2 * i) = b.v * cs;
    SL(gb.s, m.off_u + 2 * i + 1) = b.v * sn;
    neg |= b.v <= 0.0;
  };
  int i = i0 + r;
  for (; i + 4 < i1; i += 8) {
    const Bus b0 = load(i), b1 = load(i + 4);
    finish(i, b0);
    finish(i + 4, b1);
  }
  if (i < i1) finish(i, load(i));
  if (neg) atomicOr(&w.flags[g * kGroup + sc], 4);
}

#ifndef ACPF_MIS_UNROLL
#define ACPF_MIS_UNROLL 2  // 2.87 -> 2.75 ms per launch (4: 2.80; 64 registers: 3.1)
#endif
#ifndef ACPF_MIS_MINB
#define ACPF_MIS_MINB 16  // 32 registers, 64 resident warps/SM: 2.76 -> 2.52 ms per launch with the two-deep gathers (round 1, one-deep: 12 beat 16)
#endif
__global__ void __launch_bounds__(128, ACPF_MIS_MINB) nr_mismatch_kernel(NrDeviceModel m, NrWorkspace w) {
  const int lane = threadIdx.x & 31, r = lane >> 3, sc = lane & 7;
  const int64_t item = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int nch = (m.n_bus + kBusChunk - 1) / kBusChunk;
  const int64_t g = item / nch;
  if (g >= w.groups || !w.gactive[g]) return;
  const int i0 = (int)(item % nch) * kBusChunk, i1 = min(m.n_bus, i0 + kBusChunk);
  const GroupBase gb = group_base(m, w, g, sc);
  // the scalar region is read-only here (only block elements are written), so
  // gathers go through the non-coherent path
  const double* __restrict__ su = gb.s + m.off_u * kGroup;  // u_j: su[2j*8], su[(2j+1)*8]
  double* __restrict__ blk = gb.b;
  auto ld2 = [](const double* __restrict__ base, int j) {
    return make_double2(__ldg(base + (size_t)(2 * j) * kGroup), __ldg(base + (size_t)(2 * j + 1) * kGroup));
  };
  double fmx = 0.0;
  int bad = 0;  // bit0 NaN, bit1 Inf
  const bool s0 = m.sh_s0 != nullptr && *w.kstep == 0;
  for (int i = i0 + r; i < i1; i += 4) {
    const int p = __ldg(m.bus_row + i);
    if (p < 0) continue;  // slack: no equations
    double2 sv;
    if (s0) {
      sv = __ldg(m.sh_s0 + i);  // step 0: every scenario sits at the flat start
    } else {
      double2 acc = make_double2(0.0, 0.0);
      const int e1 = __ldg(m.y_rowptr + i + 1);
      int e = __ldg(m.y_rowptr + i);
#if ACPF_MIS_UNROLL > 1
      // ACPF_MIS_UNROLL gathers in flight, summed in order (same rounding)
      for (; e + ACPF_MIS_UNROLL <= e1; e += ACPF_MIS_UNROLL) {
        int c[ACPF_MIS_UNROLL];
        double2 y[ACPF_MIS_UNROLL], uj[ACPF_MIS_UNROLL];
#pragma unroll
        for (int k = 0; k < ACPF_MIS_UNROLL; ++k) c[k] = __ldg(m.y_col + e + k);
#pragma unroll
        for (int k = 0; k < ACPF_MIS_UNROLL; ++k) y[k] = __ldg(m.y_val + e + k), uj[k] = ld2(su, c[k]);
#pragma unroll
        for (int k = 0; k < ACPF_MIS_UNROLL; ++k) {
          acc.x += y[k].x * uj[k].x - y[k].y * uj[k].y;
          acc.y += y[k].x * uj[k].y + y[k].y * uj[k].x;
        }
      }
#endif
      for (; e < e1; ++e) {
        const double2 y = __ldg(m.y_val + e);
        const double2 uj = ld2(su, __ldg(m.y_col + e));
        acc.x += y.x * uj.x - y.y * uj.y;
        acc.y += y.x * uj.y + y.y * uj.x;
      }
      sv = mul_conj(ld2(su, i), acc);  // S_i = u_i conj(I_i)
    }
    const bool pq = __ldg(m.qidx + i) >= 0;
    const double fp = sv.x - __ldg(gb.s + (m.off_spec + 2 * p) * kGroup);
    bad |= isnan(fp) ? 1 : (isinf(fp) ? 2 : 0);
    fmx = fmx < fabs(fp) ? fabs(fp) : fmx;
    double fq = 0.0;
    if (pq) {
      fq = sv.y - __ldg(gb.s + (m.off_spec + 2 * p + 1) * kGroup);
      bad |= isnan(fq) ? 1 : (isinf(fq) ? 2 : 0);
      fmx = fmx < fabs(fq) ? fabs(fq) : fmx;
    }
    *reinterpret_cast<double2*>(&BL(blk, m.off_yx + p, 0)) = make_double2(-fp, -fq);
  }
  const int64_t s = g * kGroup + sc;
  // fmax of non-negative doubles is the max of their bit patterns
  if (fmx > 0.0) atomicMax(&w.fmax_bits[s], (unsigned long long)__double_as_longlong(fmx));
  if (bad) atomicOr(&w.flags[s], bad);
}

// Jacobian 2x2 blocks of every Ybus entry (i, j) straight into their LU slots,
// for the groups still active after the exit checks (first kernel of a step's
// body, so the final mismatch pass of a solve assembles nothing):
//   dS_i/dth_j = -j u_i conj(y u_j)  (j != i);  dS_i/dth_i = j u_i conj(I_i - y u_i)
//   dS_i/dV_j  =  u_i conj(y E_j) [+ conj(I_i) E_i if j == i]
//   [[H, N], [M, L]] = [[Re dS/dth, Re dS/dV], [Im dS/dth, Im dS/dV]]
// with the PV padding rows/columns of the identity equation dV = 0
// (dense_jacobian, transmission.py:383-407). I_i = sum_j Y_ij u_j is
// accumulated over the same assembly list (the Ybus row in order, slack
// columns included), the diagonal block written after the row.
// 1 / V_j for the dV terms: gathered (default) or |u_j| recomputed (ACPF_EXP_VABS)
#ifdef ACPF_EXP_VABS
#define ACPF_INV_V(uv, j) (1.0 / sqrt((uv).x * (uv).x + (uv).y * (uv).y))
#else
#define ACPF_INV_V(uv, j) (1.0 / __ldg(svm + (size_t)(j) * kGroup))
#endif
#ifndef ACPF_JAC_MINB
#define ACPF_JAC_MINB 8
#endif
#ifndef ACPF_JAC_UNROLL
#define ACPF_JAC_UNROLL 2
#endif
__global__ void __launch_bounds__(128, ACPF_JAC_MINB) nr_jacobian_kernel(NrDeviceModel m, NrWorkspace w) {
  const int lane = threadIdx.x & 31, r = lane >> 3, sc = lane & 7;
  const int64_t item = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int nch = (m.n_bus + kBusChunk - 1) / kBusChunk;
  const int64_t g = item / nch;
  if (g >= w.groups || !w.gactive[g]) return;
  const int i0 = (int)(item % nch) * kBusChunk, i1 = min(m.n_bus, i0 + kBusChunk);
  const GroupBase gb = group_base(m, w, g, sc);
  const double* __restrict__ su = gb.s + m.off_u * kGroup;
  const double* __restrict__ svm = gb.s + m.off_vm * kGroup;  // V_j: svm[j*8]
  double* __restrict__ blk = gb.b;
  auto ld2 = [](const double* __restrict__ base, int j) {
    return make_double2(__ldg(base + (size_t)(2 * j) * kGroup), __ldg(base + (size_t)(2 * j + 1) * kGroup));
  };
  // column-major [[H, N], [M, L]]: H (0,0)->0, M (1,0)->1, N (0,1)->2, L (1,1)->3;
  // one 16-byte store per block column (entries (0, j), (1, j) are adjacent)
  auto put = [&](int slot, double2 dth, double2 dv, bool pq, bool pqj, bool diag) {
    double2* const col = reinterpret_cast<double2*>(&BL(blk, m.off_lu + slot, 0));
    col[0] = make_double2(dth.x, pq ? dth.y : 0.0);
    col[kGroup] = make_double2(pqj ? dv.x : 0.0, (pq && pqj) ? dv.y : (diag ? 1.0 : 0.0));
  };
  for (int i = i0 + r; i < i1; i += 4) {
    if (__ldg(m.bus_row + i) < 0) continue;  // slack: no equations
    const double2 u = ld2(su, i);
    const bool pq = __ldg(m.qidx + i) >= 0;
    double2 acc = make_double2(0.0, 0.0);
    int dslot = -1;
    double2 dy = make_double2(0.0, 0.0);
    const int a0 = __ldg(m.asm_ptr + i), a1 = __ldg(m.asm_ptr + i + 1);
    // one assembly entry: I_i accumulation, then the off-diagonal block
    auto entry = [&](int slot, double2 y, int jb, double2 uj, double vj, int qj) {
      acc.x += y.x * uj.x - y.y * uj.y;
      acc.y += y.x * uj.y + y.y * uj.x;
      if (jb == i) {
        dslot = slot;
        dy = y;
        return;
      }
      if (slot < 0) return;  // slack column
      // u_i conj(y E_j) = u_i conj(y u_j) / V_j (V_j real): no E gather
      const double2 wt = mul_conj(u, cmul(y, uj));
      const double rv = 1.0 / vj;
      const double2 wv = make_double2(wt.x * rv, wt.y * rv);
      put(slot, make_double2(wt.y, -wt.x), wv, pq, qj >= 0, false);
    };
    // ACPF_JAC_UNROLL entries' gathers (u_j, V_j) in flight before any is
    // used: the kernel waits on these loads (long_scoreboard); same
    // arithmetic order as one entry at a time
    int a = a0;
    constexpr int U = ACPF_JAC_UNROLL;
    for (; a + U <= a1; a += U) {
      int sl[U], jj[U], qq[U];
      double2 yy[U], uu[U];
      double vv[U];
#pragma unroll
      for (int k = 0; k < U; ++k) sl[k] = __ldg(m.asm_slot + a + k), jj[k] = __ldg(m.asm_j + a + k);
#pragma unroll
      for (int k = 0; k < U; ++k) {
        yy[k] = __ldg(m.asm_y + a + k);
        uu[k] = ld2(su, jj[k]);
        vv[k] = __ldg(svm + (size_t)jj[k] * kGroup);
        qq[k] = __ldg(m.qidx + jj[k]);
      }
#pragma unroll
      for (int k = 0; k < U; ++k) entry(sl[k], yy[k], jj[k], uu[k], vv[k], qq[k]);
    }
    for (; a < a1; ++a) {
      const int j0 = __ldg(m.asm_j + a);
      entry(__ldg(m.asm_slot + a), __ldg(m.asm_y + a), j0, ld2(su, j0), __ldg(svm + (size_t)j0 * kGroup),
            __ldg(m.qidx + j0));
    }
    if (dslot >= 0) {
      const double rv = ACPF_INV_V(u, i);
      const double2 ei = make_double2(u.x * rv, u.y * rv);  // E_i = u_i / V_i
      const double2 yu = cmul(dy, u);
      const double2 wv0 = mul_conj(u, yu);
      const double2 wv = make_double2(wv0.x * rv, wv0.y * rv);
      const double2 wt = mul_conj(u, make_double2(acc.x - yu.x, acc.y - yu.y));
      put(dslot, make_double2(-wt.y, wt.x),
          make_double2(wv.x + (acc.x * ei.x + acc.y * ei.y), wv.y + (acc.x * ei.y - acc.y * ei.x)), pq, pq,
          true);
    }
  }
}

__global__ void nr_check_kernel(NrWorkspace w, int64_t batch, int max_newton, double tol) {
  const int lane = threadIdx.x & 31;
  const int k = *w.kstep;
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

// Live groups of the unit: bit h set if group g0 + h exists and is active.
template <int NG>
__device__ __forceinline__ unsigned unit_live(const NrWorkspace& w, int64_t g0) {
  unsigned live = 0;
#pragma unroll
  for (int h = 0; h < NG; ++h)
    if (g0 + h < w.groups && w.gactive[g0 + h]) live |= 1u << h;
  return live;
}

// Point the pipe at the unit's arena (lane's copy source) and the CTA's ring.
template <class P>
__device__ __forceinline__ void pipe_setup(P& pp, const NrDeviceModel& m, const NrWorkspace& w, int64_t g0,
                                           unsigned live, uint32_t ring, int lane) {
  const size_t gstride = (size_t)(m.n_block * kBlk + m.n_scalar * kGroup);
  const int half = lane >> 4, chunk = lane & 15;
  const int h = P::NG == 1 ? 0 : half;
  pp.src = w.arena + (size_t)(g0 + h) * gstride + chunk * 2;
  pp.n_elem = (uint32_t)m.n_block;
  pp.cp_ok = (live >> h) & 1u;
  pp.nlive = __popc(live);
  pp.ring = ring;
  pp.wring = ring + P::kRingN * P::kSlot;
  pp.lane = lane;
}

// One elimination level: task = (run of block rows of the level, unit of NG
// scenario groups). Lane (r, sc) owns entry (i, j) = (r/2, r%2) of every
// block of scenario sc of each group of the unit; the NG groups share every
// address computation (their copies sit 256 B apart in each ring slot).
//
// gmajor (the tail level): consecutive CTAs take the ntask row tasks of one
// unit, so the non-tail U^ blocks every tail row of a group gathers are
// reused from L2 while that group's rows are in flight.
template <class P>
__global__ void __launch_bounds__(32) nr_factor_kernel(NrDeviceModel m, NrWorkspace w, int task0, int64_t units,
                                                       int ntask, int gmajor) {
  constexpr int NG = P::NG, CH = P::CH;
  constexpr int kSlot = P::kSlot;
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x, r = lane >> 3, sc = lane & 7;
  const int bi = r >> 1, bj = r & 1;
  const int64_t task = blockIdx.x;
  const int64_t g0 = (gmajor ? task / ntask : task % units) * NG;
  const int tk = task0 + (int)(gmajor ? task % ntask : task / units);
  const unsigned live = unit_live<NG>(w, g0);
  if (!live) return;
  const size_t gstride = (size_t)(m.n_block * kBlk + m.n_scalar * kGroup);
  double* const gb0 = w.arena + (size_t)g0 * gstride + 2 * sc;  // group h at + h*gstride
  const uint32_t ring = su32(smem);
  const uint32_t lbuf = ring + P::smem_bytes();
  // lbuf holds the row's L blocks row-major: entry (i, j) of scenario sc of
  // group h at lbuf + pos*kSlot + h*256 + 128*i + 16*sc + 8*j, so L[i][0..1]
  // is one 16-byte load; U[0..1][j] of a ring element is one too
  const uint32_t offL = kHalf * bi + 16 * sc;  // L[i][0], L[i][1] (row i)
  const uint32_t offU = kHalf * bj + 16 * sc;  // U[0][j], U[1][j] (column j)
  const int ce = 2 * bj + bi;                     // this lane's column-major entry
  // this lane's entry of LU element 0 of group 0 (stores index it by slot)
  double* const luw = &BL(gb0, m.off_lu, ce);
  const uint32_t lrow = lbuf + offL;
  // tail level: one row per task, listed in m.tail_trow (class order)
  const int p0 = gmajor ? m.tail_trow[tk] : m.task_row[tk];
  const int p1 = gmajor ? p0 + 1 : m.task_row[tk + 1];
  P pp;
  pipe_setup(pp, m, w, g0, live, ring, lane);
  pp.begin(m.stream, m.row_sptr[p0], m.row_sptr[p1]);
  unsigned zero = 0;
  // slot control words of the whole task (lane j holds slot tw + j), double
  // buffered so the next window's load is in flight a window ahead
  const int ts0 = m.row_slot[p0], ts1 = m.row_slot[p1];
  int tw = ts0;
  uint32_t winfo = ts0 + lane < ts1 ? m.slot_info[ts0 + lane] : 0u;
  uint32_t ninfo = ts0 + 32 + lane < ts1 ? m.slot_info[ts0 + 32 + lane] : 0u;
  int32_t wstore = ts0 + lane < ts1 ? m.slot_store[ts0 + lane] : 0;
  int32_t nstore = ts0 + 32 + lane < ts1 ? m.slot_store[ts0 + 32 + lane] : 0;
  int t = ts0;
  // control and store words of the slot about to run, fetched one slot ahead
  // (the shuffle is off the slot's critical path)
  uint32_t cur_info = __shfl_sync(kFull, winfo, 0);
  int32_t cur_store = __shfl_sync(kFull, wstore, 0);
  for (int p = p0; p < p1; ++p) {
    const int t0 = t;
    pp.ensure(pp.q);
    double yacc[NG];  // b_p[i]
    {
      const uint32_t sb = pp.slot_base(pp.q) + 16 * sc + 8 * bi;
#pragma unroll
      for (int h = 0; h < NG; ++h) yacc[h] = lds_f64(sb + h * kBlkBytes);
    }
    ++pp.q;
    double ir0[NG], ir1[NG];  // row i of inv(U_pp), set at the diagonal slot
    for (;; ++t) {
      const uint32_t info = cur_info;
      const int32_t stv = cur_store;
      if (t + 1 - tw == 32) {
        tw += 32;
        winfo = ninfo;
        wstore = nstore;
        ninfo = tw + 32 + lane < ts1 ? m.slot_info[tw + 32 + lane] : 0u;
        nstore = tw + 32 + lane < ts1 ? m.slot_store[tw + 32 + lane] : 0;
      }
      cur_info = __shfl_sync(kFull, winfo, (t + 1 - tw) & 31);
      cur_store = __shfl_sync(kFull, wstore, (t + 1 - tw) & 31);
      const int cnt = (int)(info >> 16);
      double a[NG], a2[NG], a3[NG], a4[NG];
#pragma unroll
      for (int h = 0; h < NG; ++h) a[h] = a2[h] = a3[h] = a4[h] = 0.0;
      if (!(info & kSlotFill)) {
        pp.ensure(pp.q);
        const uint32_t sb = pp.slot_base(pp.q) + kHalf * bj + 16 * sc + 8 * bi;
#pragma unroll
        for (int h = 0; h < NG; ++h) a[h] = lds_f64(sb + h * kBlkBytes);
        ++pp.q;
      }
      // block Crout updates: A_pt -= L_pm U_mt, lane owns (i, j); two
      // interleaved accumulator pairs keep four independent FMA chains
      // one pipeline stage at a time: its elements are contiguous in the ring,
      // so every address below is a base plus an immediate
      for (int q = 0; q < cnt;) {
        pp.ensure(pp.q);
        const int nb = min(cnt - q, ((pp.q | (CH - 1)) + 1) - pp.q);
        const uint32_t ub = pp.slot_base(pp.q) + offU;
        const uint32_t wb = pp.wring + ((uint32_t)pp.q % (uint32_t)P::kRingN) * 4;
#ifndef ACPF_EXP_NOCOMPUTE
#pragma unroll
        for (int k = 0; k < CH; k += 2) {
          if (k < nb) {
            const uint32_t la0 = lrow + lds_u32(wb + 4 * k);
            const bool two = k + 1 < nb;
            const uint32_t la1 = two ? lrow + lds_u32(wb + 4 * k + 4) : 0u;
#pragma unroll
            for (int h = 0; h < NG; ++h) {
              const double2 l0 = lds_f64x2(la0 + h * kBlkBytes);
              const double2 u0 = lds_f64x2(ub + k * kSlot + h * kBlkBytes);
              a[h] = fma(-l0.x, u0.x, a[h]);
              a2[h] = fma(-l0.y, u0.y, a2[h]);
              if (two) {
                const double2 l1 = lds_f64x2(la1 + h * kBlkBytes);
                const double2 u1 = lds_f64x2(ub + (k + 1) * kSlot + h * kBlkBytes);
                a3[h] = fma(-l1.x, u1.x, a3[h]);
                a4[h] = fma(-l1.y, u1.y, a4[h]);
              }
            }
          }
        }
#endif
        pp.q += nb;
        q += nb;
      }
#pragma unroll
      for (int h = 0; h < NG; ++h) a[h] = (a[h] + a3[h]) + (a2[h] + a4[h]);
      if (info & kSlotL) {
        // unit-upper form A = L^ U^ (L^ = L D, U^ = D^-1 U, D = diag(U_tt)):
        // L^_pt is the updated block itself; y_p -= L^_pt y_t
        pp.ensure(pp.q);
        const uint32_t yb = pp.slot_base(pp.q) + 16 * sc;
        const uint32_t lb = lbuf + (t - t0) * kSlot + offL + 8 * bj;
#pragma unroll
        for (int h = 0; h < NG; ++h) {
          const double l = a[h];
          sts_f64(lb + h * kBlkBytes, l);
          const double lo = __shfl_xor_sync(kFull, l, 8);  // entry (i, 1-j)
          const double li0 = bj ? lo : l, li1 = bj ? l : lo;
          const double2 yt = lds_f64x2(yb + h * kBlkBytes);
          yacc[h] = fma(-li1, yt.y, fma(-li0, yt.x, yacc[h]));
        }
        pp.q += 1;
      } else if (info & kSlotTail) {
        // tail row, tail column: A_pt minus the non-tail updates, stored raw
        // for the dense tail factorisation (nr_tail_kernel)
        const size_t st = (size_t)(uint32_t)stv * kBlk;
        ACPF_CHECK(st < (size_t)m.n_block * kBlk);
#pragma unroll
        for (int h = 0; h < NG; ++h)
          if ((live >> h) & 1u) luw[h * gstride + st] = a[h];
      } else {
        const size_t st = (size_t)(uint32_t)stv * kBlk;
#pragma unroll
        for (int h = 0; h < NG; ++h) {
          if (info & kSlotDiag) {
            // inv(U_pp), kept in registers for the row's U^ blocks and y_p
            const double a00 = __shfl_sync(kFull, a[h], sc), a01 = __shfl_sync(kFull, a[h], 8 + sc);
            const double a10 = __shfl_sync(kFull, a[h], 16 + sc), a11 = __shfl_sync(kFull, a[h], 24 + sc);
            const double det = a00 * a11 - a01 * a10;
            zero |= (det == 0.0 ? 1u : 0u) << h;
            const double rd = 1.0 / det;
            ir0[h] = bi ? -a10 * rd : a11 * rd;  // inv[i][0]
            ir1[h] = bi ? a00 * rd : -a01 * rd;  // inv[i][1]
          } else {
            // U^_pt = inv(U_pp) A'_pt: column j of A' from the other row's lane
            const double o = __shfl_xor_sync(kFull, a[h], 16);  // entry (1-i, j)
            const double c0 = bi ? o : a[h], c1 = bi ? a[h] : o;
            ACPF_CHECK(st < (size_t)m.n_block * kBlk);
            if ((live >> h) & 1u) luw[h * gstride + st] = ir0[h] * c0 + ir1[h] * c1;
          }
        }
      }
      if (info & kSlotRowEnd) {
        ++t;
        break;
      }
    }
    ACPF_CHECK(p >= 0 && p < m.n_rows);
    if (p >= m.tail_row0) {  // tail row: b_p - sum over non-tail t of L^_pt y_t, raw
#pragma unroll
      for (int h = 0; h < NG; ++h)
        if (bj == 0 && ((live >> h) & 1u)) BL(gb0 + h * gstride, m.off_yx + p, bi) = yacc[h];
    } else {
#pragma unroll
      for (int h = 0; h < NG; ++h) {  // y_p = inv(U_pp) (b_p - sum_t L^_pt y_t)
        const double o = __shfl_xor_sync(kFull, yacc[h], 16);  // the other row
        const double y = ir0[h] * (bi ? o : yacc[h]) + ir1[h] * (bi ? yacc[h] : o);
        if (bj == 0 && ((live >> h) & 1u)) BL(gb0 + h * gstride, m.off_yx + p, bi) = y;
      }
    }
    __syncwarp();  // lbuf of this row complete before the next row of the task reuses it
  }
  pp.finish();
  zero &= live;
  if (zero && r == 0) {
#pragma unroll
    for (int h = 0; h < NG; ++h)
      if ((zero >> h) & 1u) atomicOr(&w.flags[(g0 + h) * kGroup + sc], 8);
  }
}

// One back-substitution level: task = (run of back rows of the level, unit of NG groups).
template <class P>
__global__ void __launch_bounds__(32) nr_back_kernel(NrDeviceModel m, NrWorkspace w, int task0, int64_t units) {
  constexpr int NG = P::NG;
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x, r = lane >> 3, sc = lane & 7;
  const int bi = r >> 1, bj = r & 1;
  const int64_t task = blockIdx.x;
  const int64_t g0 = (task % units) * NG;
  const int tk = task0 + (int)(task / units);
  const unsigned live = unit_live<NG>(w, g0);
  if (!live) return;
  const size_t gstride = (size_t)(m.n_block * kBlk + m.n_scalar * kGroup);
  double* const gb0 = w.arena + (size_t)g0 * gstride + 2 * sc;
  const int r0 = m.btask_row[tk], r1 = m.btask_row[tk + 1];
  P pp;
  pipe_setup(pp, m, w, g0, live, su32(smem), lane);
  pp.begin(m.stream, m.brow_sptr[r0], m.brow_sptr[r1]);
  // back-row words of the task (lane j holds row rw + j), double buffered
  int rw = r0;
  uint32_t wrow = r0 + lane < r1 ? m.brow[r0 + lane] : 0u;
  uint32_t nrow = r0 + 32 + lane < r1 ? m.brow[r0 + 32 + lane] : 0u;
  const uint32_t offY = 16 * sc + 8 * bi;  // y[i]
  const uint32_t offUp = kHalf * bj + 16 * sc + 8 * bi, offX = 16 * sc + 8 * bj;
  for (int rr = r0; rr < r1; ++rr) {
    if (rr - rw == 32) {
      rw += 32;
      wrow = nrow;
      nrow = rw + 32 + lane < r1 ? m.brow[rw + 32 + lane] : 0u;
    }
    const uint32_t b = __shfl_sync(kFull, wrow, rr - rw);
    const int p = (int)(b & 0xfffffu);
    const int cnt = (int)(b >> 20);
    pp.ensure(pp.q);
    double yi[NG], part[NG], part2[NG];
    {
      const uint32_t yb = pp.slot_base(pp.q) + offY;
#pragma unroll
      for (int h = 0; h < NG; ++h) {
        yi[h] = lds_f64(yb + h * kBlkBytes);
        part[h] = part2[h] = 0.0;  // sum_c U^_pc[i][j] x_c[j]
      }
    }
    pp.q += 1;
    for (int q = 0; q < cnt;) {
      pp.ensure(pp.q + 1);
      const int nb = min(cnt - q, (pp.ready_upto - pp.q) >> 1);
      int k = 0;
      for (; k + 1 < nb; k += 2) {
        const int e = pp.q + 2 * k;
        const uint32_t u0 = pp.slot_base(e) + offUp, x0 = pp.slot_base(e + 1) + offX;
        const uint32_t u1 = pp.slot_base(e + 2) + offUp, x1 = pp.slot_base(e + 3) + offX;
#pragma unroll
        for (int h = 0; h < NG; ++h) {
          part[h] = fma(lds_f64(u0 + h * kBlkBytes), lds_f64(x0 + h * kBlkBytes), part[h]);
          part2[h] = fma(lds_f64(u1 + h * kBlkBytes), lds_f64(x1 + h * kBlkBytes), part2[h]);
        }
      }
      if (k < nb) {
        const int e = pp.q + 2 * k;
        const uint32_t u0 = pp.slot_base(e) + offUp, x0 = pp.slot_base(e + 1) + offX;
#pragma unroll
        for (int h = 0; h < NG; ++h)
          part[h] = fma(lds_f64(u0 + h * kBlkBytes), lds_f64(x0 + h * kBlkBytes), part[h]);
      }
      pp.q += 2 * nb;
      q += nb;
    }
#pragma unroll
    for (int h = 0; h < NG; ++h) {
      const double pt = part[h] + part2[h];
      const double po = __shfl_xor_sync(kFull, pt, 8);
      const double x = yi[h] - (bj ? po + pt : pt + po);  // x_p[i] = (y_p - sum_c U^_pc x_c)[i]
      if (bj == 0 && ((live >> h) & 1u)) BL(gb0 + h * gstride, m.off_yx + p, bi) = x;
    }
  }
  pp.finish();
}

// scenarios whose factorisation hit an exact zero pivot stop here (state not
// updated): status, iteration count, and out of the active set before the
// next step's phasor applies the corrections
__global__ void nr_zero_pivot_kernel(NrWorkspace w, int64_t batch) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= batch || !w.active[s]) return;
  if (w.flags[s] & 8) {
    w.status[s] = ACPF_NR_ZERO_PIVOT;
    w.iters[s] = *w.kstep;
    w.active[s] = 0;
  }
}

__global__ void nr_step_advance_kernel(NrWorkspace w) { *w.kstep += 1; }

// device-side Newton loop (conditional graph nodes): continue while any
// scenario is active after the exit checks
__global__ void nr_cond_kernel(const int* n_active, cudaGraphConditionalHandle a, cudaGraphConditionalHandle b) {
  const unsigned go = *n_active > 0 ? 1u : 0u;
  cudaGraphSetConditional(a, go);
  cudaGraphSetConditional(b, go);
}

// kernels the device loop launched in this solve (heads = bodies + 1)
__global__ void nr_count_kernel(NrWorkspace w, int n_head, int n_body, int n_body0, int shared0) {
  const int k = *w.kstep;
  const int bodies = shared0 && k > 0 ? n_body0 + (k - 1) * n_body : k * n_body;
  w.kstep[1] += 1 + (k + 1) * n_head + bodies + 1 + 1;  // init, heads, bodies, output, this kernel
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

// First Newton step with the LU of the flat-start Jacobian, which is the same
// for every scenario (nr_flat_start_factor, computed once per plan): one warp
// per scenario group runs the whole forward substitution (y_p = inv(D_p)
// (b_p - sum_t L^_pt y_t)) and back substitution (x_p = y_p - sum_c U^_pc x_c)
// over the rows in elimination order. The factors are read-only and shared by
// every group (32 B per slot, L2-resident); only the group's y/x elements are
// read and written. Lane = (half, sc, i): the two half-warps take alternate
// slots of each row, lane pair (sc, 0/1) the two entries of scenario sc.
__global__ void __launch_bounds__(128) nr_shared_step_kernel(NrDeviceModel m, NrWorkspace w) {
  const int lane = threadIdx.x & 31, half = lane >> 4, sc = (lane >> 1) & 7, i = lane & 1;
  const int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (g >= w.groups || !w.gactive[g]) return;
  double* const yx = w.arena + (size_t)g * (m.n_block * kBlk + m.n_scalar * kGroup) +
                     (size_t)m.off_yx * kBlk + 2 * sc;
  const double2* __restrict__ rows = reinterpret_cast<const double2*>(m.sh_vals);  // row i of slot t: [2t + i]
  for (int p = 0; p < m.n_rows; ++p) {
    const int t0 = __ldg(m.row_slot + p), td = __ldg(m.sh_diag + p);
    double acc = half ? 0.0 : yx[(size_t)p * kBlk + i];
    // this half's slots t, t + 2 loaded together (the row is a chain of
    // dependent index -> value loads); the sum keeps its order
    int t = t0 + half;
    for (; t + 2 < td; t += 4) {
      const int c0 = __ldg(m.sh_col + t), c1 = __ldg(m.sh_col + t + 2);
      const double2 l0 = __ldg(rows + 2 * t + i), l1 = __ldg(rows + 2 * (t + 2) + i);
      const double2 y0 = *reinterpret_cast<const double2*>(yx + (size_t)c0 * kBlk);
      const double2 y1 = *reinterpret_cast<const double2*>(yx + (size_t)c1 * kBlk);
      acc = fma(-l0.y, y0.y, fma(-l0.x, y0.x, acc));
      acc = fma(-l1.y, y1.y, fma(-l1.x, y1.x, acc));
    }
    if (t < td) {
      const int c = __ldg(m.sh_col + t);
      const double2 l = __ldg(rows + 2 * t + i);
      const double2 y = *reinterpret_cast<const double2*>(yx + (size_t)c * kBlk);
      acc = fma(-l.y, y.y, fma(-l.x, y.x, acc));
    }
    acc += __shfl_xor_sync(kFull, acc, 16);
    const double o = __shfl_xor_sync(kFull, acc, 1);
    const double2 d = __ldg(rows + 2 * td + i);  // row i of inv(D_p)
    const double y = d.x * (i ? o : acc) + d.y * (i ? acc : o);
    if (!half) yx[(size_t)p * kBlk + i] = y;
    __syncwarp();
  }
  for (int p = m.n_rows - 1; p >= 0; --p) {
    const int td = __ldg(m.sh_diag + p), t1 = __ldg(m.row_slot + p + 1);
    double part = 0.0;
    int t = td + 1 + half;
    for (; t + 2 < t1; t += 4) {
      const int c0 = __ldg(m.sh_col + t), c1 = __ldg(m.sh_col + t + 2);
      const double2 u0 = __ldg(rows + 2 * t + i), u1 = __ldg(rows + 2 * (t + 2) + i);
      const double2 x0 = *reinterpret_cast<const double2*>(yx + (size_t)c0 * kBlk);
      const double2 x1 = *reinterpret_cast<const double2*>(yx + (size_t)c1 * kBlk);
      part = fma(u0.y, x0.y, fma(u0.x, x0.x, part));
      part = fma(u1.y, x1.y, fma(u1.x, x1.x, part));
    }
    if (t < t1) {
      const int c = __ldg(m.sh_col + t);
      const double2 u = __ldg(rows + 2 * t + i);
      const double2 x = *reinterpret_cast<const double2*>(yx + (size_t)c * kBlk);
      part = fma(u.y, x.y, fma(u.x, x.x, part));
    }
    part += __shfl_xor_sync(kFull, part, 16);
    if (!half) yx[(size_t)p * kBlk + i] -= part;
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// Dense tail: on-chip LU of the top of the elimination tree (FP64 DMMA)
// ---------------------------------------------------------------------------
//
// The last T block rows of the level-sorted order (NrSchedule::tail_*; for
// gb2224 the 62 single-row "chain" levels plus one 2-row level: 64 rows,
// 2,332+ of the 4,096 blocks filled, 49% of all Crout updates) have almost no
// parallelism left in the sparse schedule: each level is one row and every
// row re-gathers the U^ rows of all earlier tail rows from HBM. Instead, the
// tail level of nr_factor_kernel applies only the updates from non-tail rows
// (all tail rows in parallel) and stores the partial blocks raw; this kernel
// then finishes the block LU of the 2T x 2T matrix (2T <= 128) per scenario
// entirely on chip, right-looking in the same unit-upper 2x2-block form
// (A = L^ U^, L^_kk = D_k, U^ = D^-1 U), with the right-hand side carried as
// an extra column (forward substitution), followed by the back substitution.
// The tail's U^ never goes to HBM; only x of the tail rows is written, and
// the non-tail back substitution reads it like any other x_c.
//
// One CTA per scenario, 16 warps; warp w keeps scalar rows 8w..8w+7 of the
// whole matrix (17 column tiles of 8, tile 16 = the right-hand side at column
// 128) in registers as mma.m8n8k4.f64 accumulator fragments. Per panel of 8
// scalar columns (4 block columns):
//   (a) the panel column and the panel rows go to shared memory;
//   (b) one warp factors the 8 x 8 diagonal block (4 block steps: D^-1, U^,
//       update) - L^11, D^-1, U^11;
//   (c) the panel rows' U^ blocks right of the panel and their y (one thread
//       per column: forward substitution with L^11, D^-1) and the L^ blocks
//       of the rows below (one thread per row: forward with U^11);
//   (d) every warp below the panel updates its accumulators with two DMMAs
//       per column tile: C -= L^(rows, panel) U^(panel, columns).
// Pivot blocks are checked for exact zero like the sparse kernel (flag 8).
constexpr int kTW = 2 * kTailMaxRows / 8;  // warps: one 8-row strip each
constexpr int kTRows = 2 * kTailMaxRows;  // 128 scalar rows
constexpr int kTYCol = kTRows;    // the right-hand side column
constexpr int kTTiles = kTRows / 8 + 1;
// U row stride >= 8 kTTiles, = 4 (mod 16): conflict-free B fragments (4 rows x 8 cols)
constexpr int kTLd = ((8 * (2 * kTailMaxRows / 8 + 1) + 11) / 16) * 16 + 4;
constexpr int kTPcLd = 12;        // panel-column stride: conflict-free A fragments (8 rows x 4 cols)
// (c): threads [0, kTColThreads) solve the panel row's columns (at most
// kTRows - 8 plus y), the rest the rows below the panel (at most kTRows - 8)
constexpr int kTColThreads = ((kTRows - 7 + 31) / 32) * 32;
static_assert(kTW * 32 - kTColThreads >= kTRows - 8, "dense tail: too few threads for the panel solves");
constexpr size_t kTailSmem = ((size_t)kTRows * kTLd + (size_t)kTRows * kTPcLd + 16 * 16 + 2 * kTRows) * 8 + 16;

__device__ __forceinline__ void dmma_t(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// Panel-specialised pieces of nr_tail_kernel: with the panel index a template
// constant every accumulator tile index is static, so the tile loops carry no
// predicates or warp syncs and the B-fragment loads can be scheduled ahead of
// the DMMAs (the runtime-indexed form ran the update phase at 1/5 of the DMMA
// pipe rate). Tiles past the matrix are zero and stay zero.
// (d) for panel P: C -= L^(strip, panel) U^(panel, tiles right of it). The
// next panel's owner updates its diagonal tile first and publishes it (look-
// ahead: warp 0 factors it while the other warps are still updating).
template <int P>
__device__ __forceinline__ void tail_update(double (&C)[kTTiles][2], const double* Pc, double* U, int crow,
                                            int ccol, int lane, bool owner, volatile int* ready) {
  const double a0 = -Pc[crow * kTPcLd + (lane & 3)], a1 = -Pc[crow * kTPcLd + 4 + (lane & 3)];
  const double* const ub0 = U + (8 * P + (lane & 3)) * kTLd + (lane >> 2);
  const double* const ub1 = ub0 + 4 * kTLd;
  if (P + 1 < kTTiles && owner) {
    dmma_t(C[P + 1][0], C[P + 1][1], a0, ub0[8 * (P + 1)]);
    dmma_t(C[P + 1][0], C[P + 1][1], a1, ub1[8 * (P + 1)]);
    *reinterpret_cast<double2*>(U + crow * kTLd + 8 * (P + 1) + ccol) = make_double2(C[P + 1][0], C[P + 1][1]);
    __threadfence_block();
    __syncwarp();
    if (lane == 0) *ready = P + 1;
  }
  const int jd = owner ? P + 2 : P + 1;  // first tile still to update
  double b[kTTiles];
#pragma unroll
  for (int j = P + 1; j < kTTiles; ++j) b[j] = ub0[8 * j];
#pragma unroll
  for (int j = P + 1; j < kTTiles; ++j)
    if (j >= jd) dmma_t(C[j][0], C[j][1], a0, b[j]);
#pragma unroll
  for (int j = P + 1; j < kTTiles; ++j) b[j] = ub1[8 * j];
#pragma unroll
  for (int j = P + 1; j < kTTiles; ++j)
    if (j >= jd) dmma_t(C[j][0], C[j][1], a1, b[j]);
}

// (a) for panel P: the panel column -> Pc; the owner's strip right of its
// (already factored) diagonal tile -> U
template <int P>
__device__ __forceinline__ void tail_store_panel(const double (&C)[kTTiles][2], double* Pc, double* U, int crow,
                                                 int ccol, bool owner) {
  *reinterpret_cast<double2*>(Pc + crow * kTPcLd + ccol) = make_double2(C[P][0], C[P][1]);
  if (owner) {
#pragma unroll
    for (int j = P + 1; j < kTTiles; ++j)
      *reinterpret_cast<double2*>(U + crow * kTLd + 8 * j + ccol) = make_double2(C[j][0], C[j][1]);
  }
}

// (b) the 8 x 8 diagonal block of a panel (4 x 4 blocks of 2 x 2) in shared
// memory, 4 block steps by one warp: pivot inverses D_k^-1 -> dinv, U^ blocks
// right of each pivot, update of the blocks below; leaves L^11 (lower), D
// (diagonal, raw) and U^11 (upper) in place. r0: first scalar row of the panel.
__device__ __forceinline__ void tail_diag_block(double* Dg, double* dinv, int lane, int r0, int n2, int* zflag) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double a00 = Dg[(2 * k) * kTLd + 2 * k], a01 = Dg[(2 * k) * kTLd + 2 * k + 1];
    const double a10 = Dg[(2 * k + 1) * kTLd + 2 * k], a11 = Dg[(2 * k + 1) * kTLd + 2 * k + 1];
    const double det = a00 * a11 - a01 * a10;
    const double rd = 1.0 / det;
    const double i00 = a11 * rd, i01 = -a01 * rd, i10 = -a10 * rd, i11 = a00 * rd;
    if (lane == 0) {
      dinv[4 * k] = i00;
      dinv[4 * k + 1] = i01;
      dinv[4 * k + 2] = i10;
      dinv[4 * k + 3] = i11;
      if (det == 0.0 && r0 + 2 * k < n2) *zflag = 1;
    }
    // U^ blocks (k, mb), mb = k+1..3: lanes 0 .. 4(3-k)-1, one entry each
    const int nu = 4 * (3 - k);
    double u = 0.0;
    int ui = 0, uc = 0;
    if (lane < nu) {
      ui = (lane & 3) >> 1;
      uc = 2 * (k + 1 + (lane >> 2)) + (lane & 1);
      const double f0 = Dg[(2 * k) * kTLd + uc], f1 = Dg[(2 * k + 1) * kTLd + uc];
      u = ui ? i10 * f0 + i11 * f1 : i00 * f0 + i01 * f1;
    }
    __syncwarp();
    if (lane < nu) Dg[(2 * k + ui) * kTLd + uc] = u;
    __syncwarp();
    // trailing entries of the block: F(ri, ci) -= L^(ri, 2k..) U^(2k.., ci)
    const int nr = 6 - 2 * k;
    for (int e = lane; e < nr * nr; e += 32) {
      const int ri = 2 * k + 2 + e / nr, ci = 2 * k + 2 + e % nr;
      Dg[ri * kTLd + ci] -= Dg[ri * kTLd + 2 * k] * Dg[(2 * k) * kTLd + ci] +
                            Dg[ri * kTLd + 2 * k + 1] * Dg[(2 * k + 1) * kTLd + ci];
    }
    __syncwarp();
  }
}

// panel index -> template constant (panels 0 .. kTW-1; a panel past the tail's
// tiles maps to the last one and never runs)
#define ACPF_TAIL_PANEL_CASE(P, CALL) \
  case P:                              \
    CALL((P < kTW ? P : kTW - 1));     \
    break;
#define ACPF_TAIL_PANEL_SWITCH(p, CALL)                                                           \
  switch (p) {                                                                                    \
    ACPF_TAIL_PANEL_CASE(0, CALL) ACPF_TAIL_PANEL_CASE(1, CALL) ACPF_TAIL_PANEL_CASE(2, CALL)     \
    ACPF_TAIL_PANEL_CASE(3, CALL) ACPF_TAIL_PANEL_CASE(4, CALL) ACPF_TAIL_PANEL_CASE(5, CALL)     \
    ACPF_TAIL_PANEL_CASE(6, CALL) ACPF_TAIL_PANEL_CASE(7, CALL) ACPF_TAIL_PANEL_CASE(8, CALL)     \
    ACPF_TAIL_PANEL_CASE(9, CALL) ACPF_TAIL_PANEL_CASE(10, CALL) ACPF_TAIL_PANEL_CASE(11, CALL)   \
    ACPF_TAIL_PANEL_CASE(12, CALL) ACPF_TAIL_PANEL_CASE(13, CALL) ACPF_TAIL_PANEL_CASE(14, CALL)  \
    default:                                                                                      \
      CALL((15 < kTW ? 15 : kTW - 1));                                                            \
      break;                                                                                      \
  }

#ifndef ACPF_TAIL_MINB
#define ACPF_TAIL_MINB (kTailMaxRows <= 48 ? 2 : 1)  // CTAs per SM the register budget must allow
#endif
__global__ void __launch_bounds__(kTW * 32, ACPF_TAIL_MINB) nr_tail_kernel(NrDeviceModel m, NrWorkspace w) {
  extern __shared__ __align__(16) double tsm[];
  double* const U = tsm;                  // [kTRows][kTLd]
  double* const Pc = U + kTRows * kTLd;   // [kTRows][kTPcLd]
  double* const Dv = Pc + kTRows * kTPcLd;  // [16 panels][4][2x2] pivot inverses
  double* const xs = Dv + 16 * 16;        // [kTRows] solution
  int* const zflag = reinterpret_cast<int*>(xs + 2 * kTRows);
  volatile int* const ready = zflag + 1;  // last panel whose diagonal tile is in U (look-ahead)
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t s = blockIdx.x;
  const int64_t g = s / kGroup;
  const int sc = (int)(s % kGroup);
  if (g >= w.groups || !w.gactive[g] || !w.active[s]) return;
  const int T = m.tail_T, n2 = 2 * T, np = (n2 + 7) >> 3;
  const double* const gsrc = w.arena + (size_t)g * (m.n_block * kBlk + m.n_scalar * kGroup) + 2 * sc;

  // ---- load: zero, identity on the padding, scatter the tail blocks and y
  for (int i = tid; i < 8 * np * kTLd; i += kTW * 32) U[i] = 0.0;
  __syncthreads();
  for (int r = n2 + tid; r < 8 * np; r += kTW * 32) U[r * kTLd + r] = 1.0;
  for (int k = tid; k < m.n_tail_slot; k += kTW * 32) {
    const int2 e = __ldg(m.tail_slot + k);
    ACPF_CHECK(e.x >= 0 && e.x < m.n_block && e.y >= 0 && e.y < T * T);
    const double* src = gsrc + (size_t)e.x * kBlk;  // column j of the block at +16 j
    const double2 c0 = *reinterpret_cast<const double2*>(src);
    const double2 c1 = *reinterpret_cast<const double2*>(src + 2 * kGroup);
    const int i = e.y / T, j = e.y - (e.y / T) * T;
    double* d = U + (2 * i) * kTLd + 2 * j;
    d[0] = c0.x;
    d[kTLd] = c0.y;
    d[1] = c1.x;
    d[kTLd + 1] = c1.y;
  }
  for (int i = tid; i < T; i += kTW * 32) {
    const double2 y = *reinterpret_cast<const double2*>(gsrc + (size_t)(m.off_yx + m.tail_row0 + i) * kBlk);
    U[(2 * i) * kTLd + kTYCol] = y.x;
    U[(2 * i + 1) * kTLd + kTYCol] = y.y;
  }
  if (tid == 0) *zflag = 0, *ready = 0;
  __syncthreads();
  const int crow = 8 * wid + (lane >> 2), ccol = 2 * (lane & 3);
  double C[kTTiles][2];
#pragma unroll
  for (int j = 0; j < kTTiles; ++j) {
    const double2 v = *reinterpret_cast<const double2*>(U + crow * kTLd + 8 * j + ccol);
    C[j][0] = v.x;
    C[j][1] = v.y;
  }
  if (wid == 0) tail_diag_block(U, Dv, lane, 0, n2, zflag);  // panel 0's diagonal block
  __syncthreads();

  for (int p = 0; p < np; ++p) {
    const int r0 = 8 * p;
    // (a) panel column -> Pc (rows >= r0); panel rows -> U
    if (wid >= p && wid < np) {
#define ACPF_TAIL_STORE(P) tail_store_panel<P>(C, Pc, U, crow, ccol, wid == p)
      ACPF_TAIL_PANEL_SWITCH(p, ACPF_TAIL_STORE)
#undef ACPF_TAIL_STORE
    }
    __syncthreads();
    double* const Dg = U + r0 * kTLd + r0;  // L^11 | D | U^11 of the panel (factored ahead)
    const double* const Dvp = Dv + 16 * p;
    // (c) panel rows right of the panel (thread per column, incl. y) and the
    //     L^ blocks of the rows below (thread per row)
    {
      const int ncol = 8 * np - r0 - 8;
      if (tid <= ncol) {
        const int c = tid < ncol ? r0 + 8 + tid : kTYCol;
        double x[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) x[r] = Dg[r * kTLd + (c - r0)];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
#pragma unroll
          for (int mb = 0; mb < k; ++mb) {
            x[2 * k] -= Dg[(2 * k) * kTLd + 2 * mb] * x[2 * mb] + Dg[(2 * k) * kTLd + 2 * mb + 1] * x[2 * mb + 1];
            x[2 * k + 1] -=
                Dg[(2 * k + 1) * kTLd + 2 * mb] * x[2 * mb] + Dg[(2 * k + 1) * kTLd + 2 * mb + 1] * x[2 * mb + 1];
          }
          const double a = x[2 * k], b = x[2 * k + 1];
          x[2 * k] = Dvp[4 * k] * a + Dvp[4 * k + 1] * b;
          x[2 * k + 1] = Dvp[4 * k + 2] * a + Dvp[4 * k + 3] * b;
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) Dg[r * kTLd + (c - r0)] = x[r];
      }
      const int t = tid - kTColThreads;
      if (t >= 0 && t < ncol) {
        double* const row = Pc + (r0 + 8 + t) * kTPcLd;
        double x[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) x[c] = row[c];
#pragma unroll
        for (int k = 1; k < 4; ++k) {
#pragma unroll
          for (int mb = 0; mb < k; ++mb) {
            x[2 * k] -= x[2 * mb] * Dg[(2 * mb) * kTLd + 2 * k] + x[2 * mb + 1] * Dg[(2 * mb + 1) * kTLd + 2 * k];
            x[2 * k + 1] -=
                x[2 * mb] * Dg[(2 * mb) * kTLd + 2 * k + 1] + x[2 * mb + 1] * Dg[(2 * mb + 1) * kTLd + 2 * k + 1];
          }
        }
#pragma unroll
        for (int c = 0; c < 8; ++c) row[c] = x[c];
      }
    }
    __syncthreads();
    // (d) C -= L^(strip, panel) U^(panel, tiles right of the panel) on the DMMA pipe
    if (wid > p && wid < np) {
#define ACPF_TAIL_UPDATE(P) tail_update<P>(C, Pc, U, crow, ccol, lane, wid == p + 1, ready)
      ACPF_TAIL_PANEL_SWITCH(p, ACPF_TAIL_UPDATE)
#undef ACPF_TAIL_UPDATE
    } else if (wid == 0 && p + 1 < np) {
      while (*ready < p + 1) {
      }
      __threadfence_block();
      tail_diag_block(U + (r0 + 8) * kTLd + r0 + 8, Dv + 16 * (p + 1), lane, r0 + 8, n2, zflag);
    }
  }
  __syncthreads();
  // ---- back substitution x = U^-1 y (unit block upper), panel by panel from
  // the bottom: warp 0 solves the panel's 8 x 8 unit upper block, then every
  // row above subtracts the panel's contribution from its y (thread per row)
  for (int p = np - 1; p >= 0; --p) {
    const int r0 = 8 * p;
    if (wid == 0) {
      double t = lane < 8 ? U[(r0 + lane) * kTLd + kTYCol] : 0.0;
      const double* const row = U + (r0 + (lane & 7)) * kTLd + r0;
#pragma unroll
      for (int k = 3; k >= 1; --k) {
        const double x0 = __shfl_sync(kFull, t, 2 * k), x1 = __shfl_sync(kFull, t, 2 * k + 1);
        if (lane < 2 * k) t -= row[2 * k] * x0 + row[2 * k + 1] * x1;
      }
      if (lane < 8) xs[r0 + lane] = t;
    }
    __syncthreads();
    if (tid < r0) {
      double* const row = U + tid * kTLd;
      double acc = row[kTYCol];
#pragma unroll
      for (int c = 0; c < 8; ++c) acc -= row[r0 + c] * xs[r0 + c];
      row[kTYCol] = acc;
    }
    __syncthreads();
  }
  // ---- x of the tail rows -> the y/x elements (the non-tail back substitution reads them)
  double* const gdst = w.arena + (size_t)g * (m.n_block * kBlk + m.n_scalar * kGroup) + 2 * sc;
  for (int i = tid; i < T; i += kTW * 32)
    *reinterpret_cast<double2*>(gdst + (size_t)(m.off_yx + m.tail_row0 + i) * kBlk) =
        make_double2(xs[2 * i], xs[2 * i + 1]);
  if (tid == 0 && *zflag) atomicOr(&w.flags[s], 8);
}

// pipeline variants (ACPF_NR_VARIANT; measured one-step times on gb2224 x 65536
// in DESIGN.md): ring of 8 x 8 elements (6 stages in flight, ~11 warps/SM),
// 8 x 4 (2 in flight, 8 KB, ~19 warps/SM, the default) and 4 x 4
using V0 = PipeLdgsts<1, 8, 8>;
using V1 = PipeLdgsts<1, 8, 4>;
using V2 = PipeLdgsts<1, 4, 4>;
using V3 = PipeLdgsts<1, 8, 16>;  // tail level (experiment): 14 stages of 8 in flight

template <class F>
auto with_variant(int v, F&& f) {  // 3 (mixed) sizes like 1
  switch (v) {
    case 0: return f(V0{});
    case 2: return f(V2{});
    default: return f(V1{});
  }
}

}  // namespace

size_t nr_smem_bytes(int variant, int cap) {
  return with_variant(variant, [&](auto p) {
    using P = decltype(p);
    return P::smem_bytes() + (size_t)cap * P::kSlot;
  });
}

size_t nr_group_state_bytes() { return kGroup * (8 + 4 + 4 + 4 + 8 + 1) + 4; }

namespace {

template <class Q>
void launch_tail_level(const NrDeviceModel& m, const NrHostSchedule& hs, const NrWorkspace& w, int64_t groups,
                       cudaStream_t stream) {
  const int64_t units = (groups + Q::NG - 1) / Q::NG;
  for (int c = 0; c < hs.n_tail_class; ++c) {  // one launch per row-buffer class, group-major
    const int k0 = hs.tail_class_ptr[c], nt = hs.tail_class_ptr[c + 1] - k0;
    nr_factor_kernel<Q><<<(unsigned)(units * nt), 32, Q::smem_bytes() + (size_t)hs.tail_class_maxl[c] * Q::kSlot,
                          stream>>>(m, w, k0, units, nt, 1);
  }
}

template <class P>
void launch_factor_level(const NrDeviceModel& m, const NrHostSchedule& hs, const NrWorkspace& w, int64_t units,
                         int l, cudaStream_t stream) {
  if (l == hs.tail_level) {
    const int64_t groups = units * P::NG;  // the unit count of the tail's own pipe
    switch (hs.tail_variant) {
      case 0: launch_tail_level<V0>(m, hs, w, groups, stream); break;
      case 1: launch_tail_level<V1>(m, hs, w, groups, stream); break;
      case 2: launch_tail_level<V2>(m, hs, w, groups, stream); break;
      default: launch_tail_level<V3>(m, hs, w, groups, stream); break;
    }
    return;
  }
  const int k0 = hs.level_task_ptr[l], nt = hs.level_task_ptr[l + 1] - k0;
  nr_factor_kernel<P><<<(unsigned)(units * nt), 32, P::smem_bytes() + (size_t)hs.level_maxl[l] * P::kSlot, stream>>>(
      m, w, k0, units, nt, 0);
}

// mixed: levels with several tasks per group take the 4x4 ring (more
// resident warps), single-task levels (the chain) the 8x4 ring (deeper
// per-warp pipeline where the L-row buffer limits residency)
template <class P>
void launch_levels(const NrDeviceModel& m, const NrHostSchedule& hs, const NrWorkspace& w, int64_t groups,
                   cudaStream_t stream, bool mixed = false) {
  const int64_t units = (groups + P::NG - 1) / P::NG;
  for (int l = 0; l < hs.n_levels; ++l) {
    if (mixed && hs.level_task_ptr[l + 1] - hs.level_task_ptr[l] > 1)
      launch_factor_level<V2>(m, hs, w, units, l, stream);
    else
      launch_factor_level<P>(m, hs, w, units, l, stream);
  }
  if (m.tail_T > 0)
    nr_tail_kernel<<<(unsigned)(groups * kGroup), kTW * 32, kTailSmem, stream>>>(m, w);
  for (int l = 0; l < hs.n_blevels; ++l) {
    const int k0 = hs.blevel_task_ptr[l], nt = hs.blevel_task_ptr[l + 1] - k0;
    nr_back_kernel<P><<<(unsigned)(units * nt), 32, P::smem_bytes(), stream>>>(m, w, k0, units);
  }
}

}  // namespace

void NrGraphCache::release() {
  if (head) cudaGraphExecDestroy(head);
  if (body) cudaGraphExecDestroy(body);
  if (body0) cudaGraphExecDestroy(body0);
  head = body = body0 = nullptr;
  for (auto& e : solves) {
    if (e.exec) cudaGraphExecDestroy(e.exec);
    e = Solve{};
  }
  groups = batch = -1;
  arena = nullptr;
}

cudaError_t launch_nr_newton(const NrDeviceModel& m_in, const NrHostSchedule& hs, const NrWorkspace& w,
                             const NrBatchIO& io, double tol, int max_newton, cudaStream_t stream,
                             int* launches, NrGraphCache* graphs) {
  // a warm start leaves the flat start: step 0 factors per scenario and the
  // step-0 mismatch gathers phasors like every other step
  NrDeviceModel m = m_in;
  if (io.theta_start) {
    m.sh_vals = nullptr;
    m.sh_s0 = nullptr;
  }
  const int v = hs.variant;
  if (v == 3) {  // mixed: the 4x4 factor kernel is launched too
    cudaError_t e2 = cudaFuncSetAttribute(nr_factor_kernel<V2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)(V2::smem_bytes() + (size_t)hs.max_l * V2::kSlot));
    if (e2 != cudaSuccess) return e2;
  }
  cudaError_t e = with_variant(v == 3 ? 1 : v, [&](auto p) {
    using P = decltype(p);
    return cudaFuncSetAttribute(nr_factor_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(P::smem_bytes() + (size_t)hs.max_l * P::kSlot));
  });
  if (e != cudaSuccess) return e;
  if (m.tail_T > 0) {
    e = cudaFuncSetAttribute(nr_tail_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTailSmem);
    if (e != cudaSuccess) return e;
    int cap = 0;
    for (int c = 0; c < hs.n_tail_class; ++c) cap = cap > hs.tail_class_maxl[c] ? cap : hs.tail_class_maxl[c];
    auto attr = [&](auto q) {
      using Q = decltype(q);
      return cudaFuncSetAttribute(nr_factor_kernel<Q>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(Q::smem_bytes() + (size_t)cap * Q::kSlot));
    };
    e = hs.tail_variant == 0   ? attr(V0{})
        : hs.tail_variant == 1 ? attr(V1{})
        : hs.tail_variant == 2 ? attr(V2{})
                               : attr(V3{});
    if (e != cudaSuccess) return e;
  }
  const int64_t groups = (io.batch + kGroup - 1) / kGroup;
  const int nch = (m.n_bus + kBusChunk - 1) / kBusChunk;
  const int wpb = 4;
  auto blocks = [&](int64_t items) { return (unsigned)((items + wpb - 1) / wpb); };
  // one Newton step = head (phasor with the previous correction, mismatch,
  // exit checks, D2H of the active count) | host test | body (one factor
  // launch per elimination level, one back launch per back level, zero-pivot
  // bookkeeping, step counter). Kernels read the step from w.kstep, so each
  // part is step-independent and is replayed as a CUDA graph.
  auto head = [&](cudaStream_t st) -> cudaError_t {
    nr_phasor_kernel<<<blocks(groups * nch), 32 * wpb, 0, st>>>(m, w);
    nr_mismatch_kernel<<<blocks(groups * nch), 32 * wpb, 0, st>>>(m, w);
    nr_check_kernel<<<blocks(groups), 32 * wpb, 0, st>>>(w, io.batch, max_newton, tol);
    return cudaMemcpyAsync(w.host_active, w.n_active, sizeof(int), cudaMemcpyDeviceToHost, st);
  };
  auto body = [&](cudaStream_t st) -> cudaError_t {
    nr_jacobian_kernel<<<blocks(groups * nch), 32 * wpb, 0, st>>>(m, w);
    if (v == 3)
      launch_levels<V1>(m, hs, w, groups, st, true);
    else
      with_variant(v, [&](auto p) { launch_levels<decltype(p)>(m, hs, w, groups, st); });
    nr_zero_pivot_kernel<<<(unsigned)((io.batch + 255) / 256), 256, 0, st>>>(w, io.batch);
    nr_step_advance_kernel<<<1, 1, 0, st>>>(w);
    return cudaGetLastError();
  };
  // step 0 with the shared flat-start LU: no factorisation, one launch of
  // substitutions per group (the zero-pivot case was excluded on the host)
  const bool shared0 = m.sh_vals != nullptr;
  auto body0 = [&](cudaStream_t st) -> cudaError_t {
    nr_shared_step_kernel<<<blocks(groups), 32 * wpb, 0, st>>>(m, w);
    nr_step_advance_kernel<<<1, 1, 0, st>>>(w);
    return cudaGetLastError();
  };
  const int n_head = 3, n_body0 = 2;
  const int n_body = hs.n_levels + hs.n_blevels + 3 + (m.tail_T > 0 ? hs.n_tail_class : 0);
  // ---- device-side Newton loop: the whole solve is one graph,
  //   init -> head -> cond -> IF(active){ step-0 body } ->
  //   WHILE(active){ head -> cond -> IF(active){ body } } -> output -> count
  // so a solve makes no host round trip per Newton step (the exit test of
  // _newton_loop, transmission.py:347-359, is evaluated by nr_cond_kernel).
  static const bool devloop = [] {
    const char* v = std::getenv("ACPF_NR_DEVLOOP");
    return !(v && v[0] == '0');
  }();
  if (graphs && devloop) {
    const void* key[5] = {io.p_spec, io.q_spec, io.theta_out, io.iterations, io.theta_start};
    NrGraphCache::Solve* slot = nullptr;
    for (auto& e : graphs->solves) {
      bool hit = e.exec && e.batch == io.batch && e.tol == tol && e.max_newton == max_newton && e.arena == w.arena;
      for (int i = 0; i < 5; ++i) hit = hit && e.io[i] == key[i];
      if (hit) slot = &e;
    }
    if (!slot) {
      slot = &graphs->solves[0];  // the least recently used entry is rebuilt
      for (auto& e : graphs->solves)
        if (e.used < slot->used) slot = &e;
      if (slot->exec) cudaGraphExecDestroy(slot->exec);
      *slot = NrGraphCache::Solve{};
      bool ok = graphs->capture || cudaStreamCreateWithFlags(&graphs->capture, cudaStreamNonBlocking) == cudaSuccess;
      cudaStream_t c1 = nullptr, c2 = nullptr;
      ok = ok && cudaStreamCreateWithFlags(&c1, cudaStreamNonBlocking) == cudaSuccess &&
           cudaStreamCreateWithFlags(&c2, cudaStreamNonBlocking) == cudaSuccess;
      cudaGraph_t g = nullptr;
      const cudaStreamCaptureMode mode = cudaStreamCaptureModeThreadLocal;
      auto head_dev = [&](cudaStream_t st) {
        nr_phasor_kernel<<<blocks(groups * nch), 32 * wpb, 0, st>>>(m, w);
        nr_mismatch_kernel<<<blocks(groups * nch), 32 * wpb, 0, st>>>(m, w);
        nr_check_kernel<<<blocks(groups), 32 * wpb, 0, st>>>(w, io.batch, max_newton, tol);
      };
      // append a conditional node at the capture position of `st`; returns its body graph
      auto add_cond = [&](cudaStream_t st, cudaGraphConditionalHandle h, cudaGraphConditionalNodeType t) {
        cudaStreamCaptureStatus cs;
        cudaGraph_t cg = nullptr;
        const cudaGraphNode_t* deps = nullptr;
        size_t nd = 0;
        cudaGraph_t bodyg = nullptr;
        if (cudaStreamGetCaptureInfo(st, &cs, nullptr, &cg, &deps, &nd) != cudaSuccess) return bodyg;
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = t;
        cp.conditional.size = 1;
        cudaGraphNode_t node;
        if (cudaGraphAddNode(&node, cg, deps, nd, &cp) != cudaSuccess) return bodyg;
        if (cudaStreamUpdateCaptureDependencies(st, &node, 1, cudaStreamSetCaptureDependencies) != cudaSuccess)
          return bodyg;
        return cp.conditional.phGraph_out[0];
      };
      auto graph_of = [&](cudaStream_t st) {
        cudaStreamCaptureStatus cs;
        cudaGraph_t cg = nullptr;
        cudaStreamGetCaptureInfo(st, &cs, nullptr, &cg, nullptr, nullptr);
        return cg;
      };
      const bool shared0_ok = shared0;
      cudaGraph_t tmp = nullptr;
      if (ok) ok = cudaStreamBeginCapture(graphs->capture, mode) == cudaSuccess;
      if (ok) {
        cudaStream_t s0 = graphs->capture;
        cudaGraph_t root = graph_of(s0);
        cudaGraphConditionalHandle h_w, h_i0;
        ok = cudaGraphConditionalHandleCreate(&h_w, root, 0, cudaGraphCondAssignDefault) == cudaSuccess &&
             cudaGraphConditionalHandleCreate(&h_i0, root, 0, cudaGraphCondAssignDefault) == cudaSuccess;
        nr_init_kernel<<<blocks(groups), 32 * wpb, 0, s0>>>(m, w, io);
        head_dev(s0);
        nr_cond_kernel<<<1, 1, 0, s0>>>(w.n_active, h_i0, h_w);
        cudaGraph_t b0 = ok ? add_cond(s0, h_i0, cudaGraphCondTypeIf) : nullptr;
        ok = ok && b0;
        if (ok) {  // step 0 (shared flat-start LU, or a full factorisation)
          ok = cudaStreamBeginCaptureToGraph(c1, b0, nullptr, nullptr, 0, mode) == cudaSuccess;
          if (ok) {
            if (shared0_ok) body0(c1); else body(c1);
            ok = cudaStreamEndCapture(c1, &tmp) == cudaSuccess;
          }
        }
        cudaGraph_t wb = ok ? add_cond(s0, h_w, cudaGraphCondTypeWhile) : nullptr;
        ok = ok && wb;
        if (ok) {  // while body: head, cond, IF(active){ body }
          ok = cudaStreamBeginCaptureToGraph(c1, wb, nullptr, nullptr, 0, mode) == cudaSuccess;
          if (ok) {
            cudaGraphConditionalHandle h_i;
            ok = cudaGraphConditionalHandleCreate(&h_i, wb, 0, cudaGraphCondAssignDefault) == cudaSuccess;
            head_dev(c1);
            nr_cond_kernel<<<1, 1, 0, c1>>>(w.n_active, h_i, h_w);
            cudaGraph_t ib = ok ? add_cond(c1, h_i, cudaGraphCondTypeIf) : nullptr;
            ok = ok && ib;
            if (ok) {
              ok = cudaStreamBeginCaptureToGraph(c2, ib, nullptr, nullptr, 0, mode) == cudaSuccess;
              if (ok) {
                body(c2);
                ok = cudaStreamEndCapture(c2, &tmp) == cudaSuccess;
              }
            }
            ok = (cudaStreamEndCapture(c1, &tmp) == cudaSuccess) && ok;
          }
        }
        nr_output_kernel<<<blocks(groups * nch), 32 * wpb, 0, s0>>>(m, w, io);
        nr_count_kernel<<<1, 1, 0, s0>>>(w, n_head + 1, n_body, n_body0, shared0_ok ? 1 : 0);
        ok = (cudaStreamEndCapture(s0, &g) == cudaSuccess) && ok && g;
      }
      ok = ok && cudaGraphInstantiate(&slot->exec, g, 0) == cudaSuccess;
      if (g) cudaGraphDestroy(g);
      if (c1) cudaStreamDestroy(c1);
      if (c2) cudaStreamDestroy(c2);
      if (ok) {
        slot->batch = io.batch;
        slot->tol = tol;
        slot->max_newton = max_newton;
        slot->arena = w.arena;
        for (int i = 0; i < 5; ++i) slot->io[i] = key[i];
      } else {
        if (slot->exec) cudaGraphExecDestroy(slot->exec);
        *slot = NrGraphCache::Solve{};
        cudaGetLastError();
      }
    }
    if (slot->exec) {
      slot->used = ++graphs->tick;
      if (launches) *launches = 0;  // counted on the device (w.kstep[1])
      return cudaGraphLaunch(slot->exec, stream);
    }
  }
  bool use_graphs = graphs != nullptr;
  if (use_graphs && (graphs->groups != groups || graphs->batch != io.batch || graphs->tol != tol ||
                     graphs->max_newton != max_newton || graphs->arena != w.arena || !graphs->head ||
                     graphs->warm != (io.theta_start != nullptr))) {
    graphs->release();
    if (!graphs->capture && cudaStreamCreateWithFlags(&graphs->capture, cudaStreamNonBlocking) != cudaSuccess)
      use_graphs = false;
    auto capture = [&](auto&& seq, cudaGraphExec_t* out) -> bool {
      cudaGraph_t gr = nullptr;
      if (cudaStreamBeginCapture(graphs->capture, cudaStreamCaptureModeThreadLocal) != cudaSuccess) return false;
      const cudaError_t r = seq(graphs->capture);
      const cudaError_t r2 = cudaStreamEndCapture(graphs->capture, &gr);
      bool ok = r == cudaSuccess && r2 == cudaSuccess && gr &&
                cudaGraphInstantiate(out, gr, 0) == cudaSuccess;
      if (gr) cudaGraphDestroy(gr);
      return ok;
    };
    if (use_graphs && capture(head, &graphs->head) && capture(body, &graphs->body) &&
        (!shared0 || capture(body0, &graphs->body0))) {
      graphs->groups = groups;
      graphs->batch = io.batch;
      graphs->tol = tol;
      graphs->max_newton = max_newton;
      graphs->arena = w.arena;
      graphs->warm = io.theta_start != nullptr;
    } else {
      graphs->release();
      cudaGetLastError();
      use_graphs = false;
    }
  }
  int nl = 0;
  nr_init_kernel<<<blocks(groups), 32 * wpb, 0, stream>>>(m, w, io);
  ++nl;
  for (int k = 0; k <= max_newton; ++k) {
    e = use_graphs ? cudaGraphLaunch(graphs->head, stream) : head(stream);
    if (e != cudaSuccess) return e;
    nl += n_head;
    e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) return e;
    if (*w.host_active == 0) break;
    const bool first = shared0 && k == 0;
    if (use_graphs)
      e = cudaGraphLaunch(first ? graphs->body0 : graphs->body, stream);
    else
      e = first ? body0(stream) : body(stream);
    if (e != cudaSuccess) return e;
    nl += first ? n_body0 : n_body;
  }
  nr_output_kernel<<<blocks(groups * nch), 32 * wpb, 0, stream>>>(m, w, io);
  ++nl;
  if (launches) *launches = nl;
  return cudaGetLastError();
}

}  // namespace acpf
