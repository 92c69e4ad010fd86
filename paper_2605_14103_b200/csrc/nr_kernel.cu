// Batched polar Newton-Raphson on sm_100a, streaming-Crout formulation.
//
// Layout: one warp = one group of kGroup = 8 scenarios; each scenario owns a
// quad of lanes (lane = r*8 + sc, sub-lane r = 0..3, scenario sc = 0..7).
// Every per-scenario quantity lives in a per-group arena of "elements":
// element e of scenario sc at arena[e*8 + sc], so one element of a group is
// 64 contiguous bytes and a warp instruction touching 4 elements is four
// fully used 64-byte segments. The schedule (LU pattern, Crout updates,
// Ybus values) is shared by all groups and read as warp-uniform data.
//
// One launch runs the whole Newton loop of the reference `_newton_loop`
// (transmission.py:333-380) for its group with no host round trip:
//   A  phasors      u = V e^{j theta}                     (transmission.py:196)
//   B  mismatch     I = Y u, S = u conj(I), F, ||F||inf    (transmission.py:194-215)
//      exit checks in the reference order: non-finite -> converged ->
//      min V <= 0 -> k == max_newton                     (transmission.py:347-359)
//   C  Jacobian assembly fused into a row-by-row (Crout, dot-product form)
//      static-pivot sparse LU refactorisation with the forward substitution
//      fused in (replaces the GMRES/FD step solve, transmission.py:361-369);
//   D  back substitution, x += dx                         (transmission.py:378)
// A, B and D split buses/updates over the four sub-lanes of a scenario.
//
// C and D are driven by one precomputed *gather stream*: every operand not
// produced inside the current row (earlier U rows, pivots, y/x entries,
// phasors) is an element index in the stream. The warp prefetches the stream
// ahead of use with cp.async (LDGSTS, 8 B per lane, 4 elements per warp
// instruction) into a shared-memory ring; completion is tracked by one
// mbarrier per 32-element segment. Rows are level-sorted (same fill), so
// prefetch runs across row boundaries and only drains where a level starts.
// The Crout updates of one LU slot are split over the quad (4 partial dot
// products, combined by a fixed butterfly), and the current row's L part
// never leaves shared memory (later rows only read U), so global traffic is
// the gathers of earlier U rows plus one write per U slot.

#include "acpf_internal.cuh"

namespace acpf {

namespace {

constexpr int kNSeg = 4;                      // ring segments (kNSeg*32 elements in flight)
constexpr int kElemBytes = kGroup * 8;        // 64
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ double lds_f64(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(a) : "memory");
  return v;
}

__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
  unsigned short v;
  asm volatile("ld.shared.u16 %0, [%1];\n" : "=h"(v) : "r"(a) : "memory");
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

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "W_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra W_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(src) : "memory");
}

__device__ __forceinline__ void cp_async_arrive(uint32_t bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared.b64 [%0];\n" ::"r"(bar) : "memory");
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// u * conj(a)
__device__ __forceinline__ double2 mul_conj(double2 u, double2 a) {
  return make_double2(u.x * a.x + u.y * a.y, u.y * a.x - u.x * a.y);
}

// sum over the quad (sub-lanes r = 0..3 of one scenario), fixed order
__device__ __forceinline__ double quad_sum(double x) {
  x = x + __shfl_xor_sync(kFull, x, 8);
  x = x + __shfl_xor_sync(kFull, x, 16);
  return x;
}

// Warp-level gather streamer; every lane executes every call.
struct Streamer {
  const uint32_t* stream;  // [n_seg + 1][32]  gidx | lpos << 22
  const uint32_t* meta;    // [n_seg + 1]      len | epoch << 6
  const double* arena;     // group arena (element e, scenario sc at arena[e*8 + sc])
  uint32_t ring;           // smem [kNSeg*32 elements][8] doubles
  uint32_t rlpos;          // smem [kNSeg*32] u16
  uint32_t rlen;           // smem [kNSeg] u32
  uint32_t bar;            // smem [kNSeg] mbarriers (count 32)
  int lane, r, sc;
  int64_t n_seg;
  int64_t k_iss, iss_total;
  uint32_t winA, winB, metaA, metaB;
  int64_t k_cur, cur_total;
  int slot, off, len;
  uint32_t phase;
  int epoch;
#ifdef ACPF_PROFILE_PHASES
  long long t_wait = 0, t_issue = 0, n_wait = 0, n_issue = 0;
#endif

  __device__ __forceinline__ void preload(int64_t k, uint32_t& win, uint32_t& mt) {
    win = stream[k * 32 + lane];
    mt = meta[k];
  }

  __device__ __forceinline__ void begin_step() {
    k_iss = 0;
    k_cur = -1;
    off = len = 0;
    epoch = 0;
    preload(0, winA, metaA);
    preload(n_seg > 0 ? 1 : 0, winB, metaB);
  }

  __device__ __forceinline__ void issue_one() {
    const int s = (int)(iss_total % kNSeg);
    const int n = (int)(metaA & 63u);
    const uint32_t seg_base = ring + (uint32_t)s * 32 * kElemBytes;
    __syncwarp();
    if (lane < n)
      asm volatile("st.shared.u16 [%0], %1;\n" ::"r"(rlpos + (s * 32 + lane) * 2),
                   "h"((unsigned short)(winA >> 22))
                   : "memory");
    if (lane == 0)
      asm volatile("st.shared.u32 [%0], %1;\n" ::"r"(rlen + s * 4), "r"(n) : "memory");
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int e = 4 * j + r;
      const uint32_t w = __shfl_sync(kFull, winA, e);
      if (e < n)
        cp_async8(seg_base + (uint32_t)e * kElemBytes + sc * 8, arena + (size_t)(w & 0x3fffffu) * kGroup + sc);
    }
    cp_async_arrive(bar + s * 8);
    __syncwarp();
    ++k_iss;
    ++iss_total;
    winA = winB;
    metaA = metaB;
    const int64_t nk = k_iss + 1 <= n_seg ? k_iss + 1 : n_seg;
    preload(nk, winB, metaB);
  }

  __device__ __forceinline__ void try_issue() {
#ifdef ACPF_PROFILE_PHASES
    long long i0_ = clock64();
#endif
    while (k_iss < n_seg && (k_iss - k_cur) <= kNSeg - (k_cur >= 0 ? 1 : 0) &&
           (int)(metaA >> 6) <= epoch) {
      issue_one();
#ifdef ACPF_PROFILE_PHASES
      ++n_issue;
#endif
    }
#ifdef ACPF_PROFILE_PHASES
    t_issue += clock64() - i0_;
#endif
  }

  __device__ __forceinline__ void new_epoch(int e) {
    epoch = e;
    // rows finished so far were written by this warp's lanes with st.global;
    // make them visible to the other lanes' cp.async reads
    __syncwarp();
    __threadfence_block();
    try_issue();
  }

  __device__ __forceinline__ void advance() {
    ++k_cur;
    if (k_cur > 0) ++cur_total;
    try_issue();
    if (k_iss <= k_cur) __trap();  // schedule bug: segment never issuable
    slot = (int)(cur_total % kNSeg);
#ifdef ACPF_PROFILE_PHASES
    long long w0_ = clock64();
#endif
    mbar_wait(bar + slot * 8, (phase >> slot) & 1u);
#ifdef ACPF_PROFILE_PHASES
    t_wait += clock64() - w0_;
    ++n_wait;
#endif
    phase ^= 1u << slot;
    len = (int)lds_u32(rlen + slot * 4);
    off = 0;
  }

  __device__ __forceinline__ uint32_t elem(int o) const {
    return ring + (uint32_t)(slot * 32 + o) * kElemBytes + sc * 8;
  }

  // scalar element (all four sub-lanes read their scenario's value)
  __device__ __forceinline__ double get() {
    if (off == len) advance();
    const double v = lds_f64(elem(off));
    ++off;
    return v;
  }

  __device__ __forceinline__ void end_step() { ++cur_total; }
};

__global__ void __launch_bounds__(32, 1) nr_stream_kernel(NrDeviceModel m, NrWorkspace w, NrBatchIO io,
                                                       double tol, int max_newton) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x;
  const int r = lane >> 3, sc = lane & 7;
  const int64_t g = blockIdx.x;
  if (g >= w.groups) return;
  const int64_t s = g * kGroup + sc;
  const bool valid = s < io.batch;
  double* __restrict__ A = w.arena + (size_t)g * m.n_elem * kGroup + sc;
#define EL(e) A[(size_t)(e) * kGroup]

  const uint32_t sbase = su32(smem);
  const uint32_t ring = sbase;                                   // kNSeg*32 elements
  const uint32_t lbuf = ring + kNSeg * 32 * kElemBytes;          // cap elements
  const uint32_t bar = lbuf + (uint32_t)m.cap * kElemBytes;      // kNSeg mbarriers
  const uint32_t rlpos = bar + kNSeg * 8;                        // kNSeg*32 u16
  const uint32_t rlen = rlpos + kNSeg * 32 * 2;                  // kNSeg u32
  const uint32_t lbuf_sc = lbuf + sc * 8;
  if (lane == 0) {
    for (int k = 0; k < kNSeg; ++k) mbar_init(bar + k * 8, 32);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncwarp();

  Streamer st;
  st.stream = m.stream;
  st.meta = m.segmeta;
  st.arena = w.arena + (size_t)g * m.n_elem * kGroup;
  st.ring = ring;
  st.rlpos = rlpos;
  st.rlen = rlen;
  st.bar = bar;
  st.lane = lane;
  st.r = r;
  st.sc = sc;
  st.n_seg = m.n_seg;
  st.iss_total = 0;
  st.cur_total = 0;
  st.phase = 0;
  const bool no_spill = m.cap >= m.max_l;

  // flat start + this scenario's specified injections (buses/entries split over the quad)
  for (int i = r; i < m.n_bus; i += 4) {
    EL(m.off_th + i) = m.theta_init[i];
    EL(m.off_vm + i) = m.vmag_init[i];
  }
  for (int k = r; k < m.n_j; k += 4) {
    double v = 0.0;
    if (valid)
      v = k < m.n_theta ? io.p_spec[s * m.n_theta + k] : io.q_spec[s * m.n_q + (k - m.n_theta)];
    EL(m.off_spec + k) = v;
  }
  __syncwarp();

  bool done = !valid;
  int status = 0, iters = 0;
  double fout = 0.0;

#ifdef ACPF_PROFILE_PHASES
  long long tA = 0, tB = 0, tC = 0, tD = 0, tq;
#define PHASE_MARK(acc) do { long long now_ = clock64(); acc += now_ - tq; tq = now_; } while (0)
#else
#define PHASE_MARK(acc) do {} while (0)
#endif
  for (int k = 0; k <= max_newton; ++k) {
#ifdef ACPF_PROFILE_PHASES
    tq = clock64();
#endif
    // ---- A: phasors, min V
    double vmin = __longlong_as_double(0x7ff0000000000000LL);
    for (int i = r; i < m.n_bus; i += 4) {
      const double t = EL(m.off_th + i), v = EL(m.off_vm + i);
      double sn, cs;
      sincos(t, &sn, &cs);
      EL(m.off_e + 2 * i) = cs;
      EL(m.off_e + 2 * i + 1) = sn;
      EL(m.off_u + 2 * i) = v * cs;
      EL(m.off_u + 2 * i + 1) = v * sn;
      vmin = fmin(vmin, v);
    }
    __syncwarp();
    PHASE_MARK(tA);
    // ---- B: injections and mismatch
    double fmx = 0.0;
    int bad = 0;  // bit0 NaN, bit1 Inf
    for (int i = r; i < m.n_bus; i += 4) {
      double2 acc = make_double2(0.0, 0.0);
      const int e1 = m.y_rowptr[i + 1];
      for (int e = m.y_rowptr[i]; e < e1; ++e) {
        const double2 y = m.y_val[e];
        const int c = m.y_col[e];
        const double ur = EL(m.off_u + 2 * c), ui = EL(m.off_u + 2 * c + 1);
        acc.x += y.x * ur - y.y * ui;
        acc.y += y.x * ui + y.y * ur;
      }
      const double2 u = make_double2(EL(m.off_u + 2 * i), EL(m.off_u + 2 * i + 1));
      const double2 sv = mul_conj(u, acc);  // S_i = u_i conj(I_i)
      const int tp = m.tpos[i], qp = m.qpos[i];
      if (tp >= 0) {
        const double f = sv.x - EL(m.off_spec + tp);
        bad |= isnan(f) ? 1 : (isinf(f) ? 2 : 0);
        fmx = fmx < fabs(f) ? fabs(f) : fmx;
        EL(m.off_yx + m.ipos[tp]) = -f;
      }
      if (qp >= 0) {
        const double f = sv.y - EL(m.off_spec + qp);
        bad |= isnan(f) ? 1 : (isinf(f) ? 2 : 0);
        fmx = fmx < fabs(f) ? fabs(f) : fmx;
        EL(m.off_yx + m.ipos[qp]) = -f;
      }
      // Jacobian blocks of row bus i straight into their LU slots
      // (dense_jacobian formulas, transmission.py:383-407):
      //   dS_i/dth_j = -j u_i conj(y u_j)        (j != i)
      //   dS_i/dth_i =  j u_i conj(I_i - y u_i)
      //   dS_i/dV_j  =  u_i conj(y E_j) [+ conj(I_i) E_i if j == i]
      //   H = Re dS/dth, N = Re dS/dV, M = Im dS/dth, L = Im dS/dV
      const double2 ei = make_double2(EL(m.off_e + 2 * i), EL(m.off_e + 2 * i + 1));
      const int a1 = m.asm_ptr[i + 1];
      for (int a = m.asm_ptr[i]; a < a1; ++a) {
        const double2 y = m.asm_y[a];
        const int jb = m.asm_j[a];
        const int4 sl = m.asm_slot[a];
        const double2 uj = make_double2(EL(m.off_u + 2 * jb), EL(m.off_u + 2 * jb + 1));
        const double2 ej = make_double2(EL(m.off_e + 2 * jb), EL(m.off_e + 2 * jb + 1));
        double2 dth, dv;
        const double2 wv = mul_conj(u, cmul(y, ej));
        if (jb != i) {
          const double2 wt = mul_conj(u, cmul(y, uj));
          dth = make_double2(wt.y, -wt.x);
          dv = wv;
        } else {
          const double2 yu = cmul(y, u);
          const double2 wt = mul_conj(u, make_double2(acc.x - yu.x, acc.y - yu.y));
          dth = make_double2(-wt.y, wt.x);
          dv = make_double2(wv.x + (acc.x * ei.x + acc.y * ei.y), wv.y + (acc.x * ei.y - acc.y * ei.x));
        }
        if (sl.x >= 0) EL(m.off_lu + sl.x) = dth.x;
        if (sl.y >= 0) EL(m.off_lu + sl.y) = dv.x;
        if (sl.z >= 0) EL(m.off_lu + sl.z) = dth.y;
        if (sl.w >= 0) EL(m.off_lu + sl.w) = dv.y;
      }
    }
    // quad reductions (order independent: max / min / or)
    fmx = fmax(fmx, __shfl_xor_sync(kFull, fmx, 8));
    fmx = fmax(fmx, __shfl_xor_sync(kFull, fmx, 16));
    vmin = fmin(vmin, __shfl_xor_sync(kFull, vmin, 8));
    vmin = fmin(vmin, __shfl_xor_sync(kFull, vmin, 16));
    bad |= __shfl_xor_sync(kFull, bad, 8);
    bad |= __shfl_xor_sync(kFull, bad, 16);
    if (!done) {
      if (bad) {
        done = true;
        status = ACPF_NR_NONFINITE;
        iters = k;
        fout = (bad & 1) ? __longlong_as_double(0x7ff8000000000000LL) : fmx;
      } else if (fmx <= tol) {
        done = true;
        status = ACPF_NR_CONVERGED;
        iters = k;
        fout = fmx;
      } else if (vmin <= 0.0) {
        done = true;
        status = ACPF_NR_VMAG_LE0;
        iters = k;
        fout = fmx;
      } else if (k == max_newton) {
        done = true;
        status = ACPF_NR_MAX_ITER;
        iters = max_newton;
        fout = fmx;
      }
    }
    PHASE_MARK(tB);
    if (__all_sync(kFull, done)) break;

    // ---- C: Crout refactorisation + forward substitution
    st.begin_step();
    st.new_epoch(0);
    bool zero_pivot = false;
    int64_t t = 0;  // LU slot
    // slot control words (lane j holds slot w0 + j), double buffered
    int64_t w0 = 0;
    uint32_t winfo = lane < m.nnz_lu ? m.slot_info[lane] : 0u;
    uint32_t ninfo = 32 + lane < m.nnz_lu ? m.slot_info[32 + lane] : 0u;
    int epoch = 0;
    for (int p = 0; p < m.n_j; ++p) {
      double yacc = 0.0;
      int pos = 0;  // position within the row
      for (;;) {
        if (t - w0 == 32) {
          w0 += 32;
          winfo = ninfo;
          const int64_t nt = w0 + 32 + lane;
          if (nt < m.nnz_lu) ninfo = m.slot_info[nt];
        }
        const uint32_t info = __shfl_sync(kFull, winfo, (int)(t - w0));
        if (info & kSlotNewEpoch) st.new_epoch(++epoch);
        const int cnt = (int)(info >> 16);
        const bool lslot = info & kSlotL, fill = info & kSlotFill;
        const int head = ((info & kSlotRowStart) ? 1 : 0) + (fill ? 0 : 1);
        const int need = head + cnt + (lslot ? 2 : 0);
        double a = 0.0, inv = 0.0, yc = 0.0;
        if (need <= 32) {
          // the whole unit sits in one ring segment (schedule guarantee)
          if (need) {
            if (st.off == st.len) st.advance();
          }
          const uint32_t e0 = st.elem(st.off);
          int o = 0;
          if (info & kSlotRowStart) yacc = lds_f64(e0 + (o++) * kElemBytes);
          if (!fill) a = lds_f64(e0 + (o++) * kElemBytes);
          if (cnt) {
            const uint32_t la = rlpos + (uint32_t)(st.slot * 32 + st.off + o) * 2;
            const uint32_t ra = e0 + o * kElemBytes;
            double part = 0.0;
            if (no_spill) {
#pragma unroll 2
              for (int q = r; q < cnt; q += 4)
                part = fma(-lds_f64(lbuf_sc + lds_u16(la + 2 * q) * kElemBytes),
                           lds_f64(ra + q * kElemBytes), part);
            } else {
              for (int q = r; q < cnt; q += 4) {
                const int lp = (int)lds_u16(la + 2 * q);
                const double l = lp < m.cap ? lds_f64(lbuf_sc + lp * kElemBytes)
                                            : EL(m.off_spill + (lp - m.cap));
                part = fma(-l, lds_f64(ra + q * kElemBytes), part);
              }
            }
            a = a + quad_sum(part);
            o += cnt;
          }
          if (lslot) {
            inv = lds_f64(e0 + o * kElemBytes);
            yc = lds_f64(e0 + (o + 1) * kElemBytes);
          }
          st.off += need;
        } else {
          // long unit: generic path across segment boundaries
          if (info & kSlotRowStart) yacc = st.get();
          if (!fill) a = st.get();
          double part = 0.0;
          int rem = cnt;
          while (rem > 0) {
            if (st.off == st.len) st.advance();
            const int nb = min(rem, st.len - st.off);
            const uint32_t la = rlpos + (uint32_t)(st.slot * 32 + st.off) * 2;
            const uint32_t ra = st.elem(st.off);
            for (int q = r; q < nb; q += 4) {
              const int lp = (int)lds_u16(la + 2 * q);
              const double l = lp < m.cap ? lds_f64(lbuf_sc + lp * kElemBytes)
                                          : EL(m.off_spill + (lp - m.cap));
              part = fma(-l, lds_f64(ra + q * kElemBytes), part);
            }
            st.off += nb;
            rem -= nb;
          }
          a = a + quad_sum(part);
          if (lslot) {
            inv = st.get();
            yc = st.get();
          }
        }
        if (lslot) {
          a *= inv;
          yacc = fma(-a, yc, yacc);
          // every quad lane holds the same value: each writes it, so each
          // lane's later reads depend only on its own store
          if (pos < m.cap)
            sts_f64(lbuf_sc + pos * kElemBytes, a);
          else
            EL(m.off_spill + (pos - m.cap)) = a;
        } else {
          if (info & kSlotDiag) {
            zero_pivot |= (a == 0.0);
            if (r == 0) EL(m.off_invd + p) = 1.0 / a;
          }
          if (r == 0) EL(m.off_lu + t) = a;
        }
        ++t;
        ++pos;
        if (info & kSlotRowEnd) break;
      }
      if (r == 0) EL(m.off_yx + p) = yacc;
    }
    PHASE_MARK(tC);
    // ---- D: back substitution (rows by back level)
    st.new_epoch(m.n_levels);
    epoch = m.n_levels;
    uint32_t bwin = 0, bnext = 0;
    if (lane < m.n_j) bwin = m.brow[lane];
    if (32 + lane < m.n_j) bnext = m.brow[32 + lane];
    for (int rr = 0; rr < m.n_j; ++rr) {
      if (rr && (rr & 31) == 0) {
        bwin = bnext;
        if (rr + 32 + lane < m.n_j) bnext = m.brow[rr + 32 + lane];
      }
      const uint32_t b = __shfl_sync(kFull, bwin, rr & 31);
      if (b >> 31) st.new_epoch(++epoch);
      const int p = (int)(b & 0xfffffu);
      int rem = (int)((b >> 20) & 0x7ffu);
      double y0, inv, part = 0.0;
      const int need = 2 + 2 * rem;
      if (need <= 32) {
        if (st.off == st.len) st.advance();
        const uint32_t e0 = st.elem(st.off);
        y0 = lds_f64(e0);
        inv = lds_f64(e0 + kElemBytes);
        for (int q = r; q < rem; q += 4)
          part = fma(-lds_f64(e0 + (2 + 2 * q) * kElemBytes), lds_f64(e0 + (3 + 2 * q) * kElemBytes), part);
        st.off += need;
      } else {
        y0 = st.get();
        inv = st.get();
        while (rem > 0) {
          if (st.off == st.len) st.advance();
          const int nb = min(rem, (st.len - st.off) >> 1);
          if (nb == 0) {  // a (u, x) pair straddles two segments
            const double u = st.get();
            const double x = st.get();
            if (r == 0) part = fma(-u, x, part);
            --rem;
            continue;
          }
          const uint32_t ra = st.elem(st.off);
          for (int q = r; q < nb; q += 4)
            part = fma(-lds_f64(ra + 2 * q * kElemBytes), lds_f64(ra + (2 * q + 1) * kElemBytes), part);
          st.off += 2 * nb;
          rem -= nb;
        }
      }
      const double x = (y0 + quad_sum(part)) * inv;
      if (r == 0) EL(m.off_yx + p) = x;
    }
    st.end_step();
    __syncwarp();
    PHASE_MARK(tD);
    // per scenario: every lane of a quad saw the same pivots
    zero_pivot = zero_pivot || __shfl_xor_sync(kFull, (int)zero_pivot, 8) ||
                 __shfl_xor_sync(kFull, (int)zero_pivot, 16);
    if (!done && zero_pivot) {
      done = true;
      status = ACPF_NR_ZERO_PIVOT;
      iters = k;
      fout = fmx;
    }
    if (!done) {
      for (int i = r; i < m.n_bus; i += 4) {
        const int tp = m.tpos[i], qp = m.qpos[i];
        if (tp >= 0) EL(m.off_th + i) = EL(m.off_th + i) + EL(m.off_yx + m.ipos[tp]);
        if (qp >= 0) EL(m.off_vm + i) = EL(m.off_vm + i) + EL(m.off_yx + m.ipos[qp]);
      }
    }
    __syncwarp();
  }

#ifdef ACPF_PROFILE_PHASES
  if (g == 0 && lane == 0)
    printf("phase cycles A %lld B %lld C %lld D %lld | wait %lld (%lld) issue %lld (%lld)\n", tA, tB, tC,
           tD, st.t_wait, st.n_wait, st.t_issue, st.n_issue);
#endif
  if (!valid) return;
  for (int i = r; i < m.n_bus; i += 4) {
    io.theta_out[s * m.n_bus + i] = EL(m.off_th + i);
    io.vmag_out[s * m.n_bus + i] = EL(m.off_vm + i);
  }
  if (r == 0) {
    if (io.converged) io.converged[s] = status == ACPF_NR_CONVERGED;
    if (io.iterations) io.iterations[s] = iters;
    if (io.fnorm) io.fnorm[s] = fout;
    if (io.status) io.status[s] = status;
  }
#undef EL
}

}  // namespace

size_t nr_smem_bytes(int cap) {
  return (size_t)kNSeg * 32 * kElemBytes + (size_t)cap * kElemBytes + kNSeg * 8 + kNSeg * 32 * 2 +
         kNSeg * 4 + 16;
}

cudaError_t launch_nr_newton(const NrDeviceModel& m, const NrWorkspace& w, const NrBatchIO& io,
                             double tol, int max_newton, cudaStream_t stream) {
  const size_t smem = nr_smem_bytes(m.cap);
  cudaError_t e = cudaFuncSetAttribute(nr_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t groups = (io.batch + kGroup - 1) / kGroup;
  nr_stream_kernel<<<(unsigned)groups, 32, smem, stream>>>(m, w, io, tol, max_newton);
  return cudaGetLastError();
}

}  // namespace acpf
