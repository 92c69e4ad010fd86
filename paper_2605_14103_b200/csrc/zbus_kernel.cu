// Fused Z-Bus fixed point on sm_100a FP64 tensor cores (DMMA).
//
// Reference loop (distribution.py:653-687): v = v0; repeat
//   i = current_injection(v)                  (:573-610)
//   v = Z i + v0                              (:673, z_apply :423-425)
//   delta = | sum|v| - sum|v_prev| |  <= tol ? (:674-679)
// then the certificate ||v - (Z i(v) + v0)||inf    (:613-621).
//
// i(v) is non-zero only on the load-touched phases l, so each sweep is the
// complex GEMM  V[n x NT] = Z[:, l] (n x |l|) * I_l (|l| x NT) + v0 over a
// tile of NT scenarios, as three real GEMMs (3-multiply complex product):
//   P1 = Zr (Ir + Ii),  P2 = (Zr + Zi) Ii,  P3 = (Zi - Zr) Ir
//   Vr = P1 - P2,       Vi = P1 + P3
// on mma.sync.m8n8k4.f64 (DMMA; sm_100a has no tcgen05 kind::f64).
//
// One CTA owns a tile of NT scenarios for its whole life (all sweeps + the
// certificate), so nothing but the final v ever leaves the SM:
//   - Z[:, l] (2.4 MB for EULV, L2-resident) streams through shared memory
//     in 64-row stages by cp.async.bulk (TMA bulk engine) + mbarrier,
//     double buffered, pre-swizzled on the host into DMMA fragment order so
//     every fragment load is one conflict-free LDS.64 per lane;
//   - I_l lives in shared memory in B-fragment order, rebuilt every sweep by
//     the column-owner thread from v at the load rows (wye then delta, in
//     the reference accumulation order), with the voltage-floor checks;
//   - the epilogue adds v0, writes v of still-running scenarios, and reduces
//     |v| per column in a fixed order (deterministic; identical for every
//     column, so results do not depend on the tile position or batch size);
//   - converged scenarios freeze (their v is not overwritten), exactly like
//     the reference returning the iterate at which delta <= tol.

#include "acpf_internal.cuh"

#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>

namespace acpf {

namespace {

#ifndef ACPF_ZB_ROW_WARPS
#define ACPF_ZB_ROW_WARPS 8
#endif
// warps = kRowWarps (row slices of a 64-row block, kRowGroups 8-row DMMA groups
// each) x kColWarps column slices. Round 1 measured 8 / 16 / 32 warps at
// 1.58M / 1.66M / 1.72M EULV/s with 64-wide tiles; with 32-wide tiles 16 warps
// (kColWarps = 2, each warp two 8-column DMMA tiles, 122 registers) is the
// fastest shape at every batch size (round 2)
constexpr int kRowWarps = ACPF_ZB_ROW_WARPS;
constexpr int kRowGroups = 8 / kRowWarps;
#ifndef ACPF_ZB_COL_WARPS
#define ACPF_ZB_COL_WARPS 2  // 16 warps with 32-wide tiles (below): 141.4 -> 139.0 ms at 262,144, 3.00 -> 2.67 ms at 4,096
#endif
constexpr int kColWarps = ACPF_ZB_COL_WARPS;
constexpr int kThreads = kRowWarps * kColWarps * 32;
#ifndef ACPF_ZB_STAGE_KS
#define ACPF_ZB_STAGE_KS 16
#endif
constexpr int kMaxKsPerStage = ACPF_ZB_STAGE_KS;  // k-steps (of 4) per Z stage
#ifndef ACPF_ZB_MINB
#define ACPF_ZB_MINB 1  // CTAs per SM (persistent grid = ACPF_ZB_MINB x SMs)
#endif
// Row-block classes: the per-column sums of every pass are formed per class
// (row blocks c, c + V, c + 2V, ... for c = 0..V-1, each in order) and the V
// class partials are then added in class order. A batch too small to fill
// the GPU with tiles (fewer tiles than resident clusters) runs each tile on a
// thread-block cluster of V CTAs, CTA c streaming class c's row blocks and
// the partials combined through distributed shared memory; larger batches run
// one CTA per tile that walks the classes one after the other. Both give the
// same bits, so results stay independent of the batch size, and a small
// batch's sweeps take ~1/V of the time.
#ifndef ACPF_ZB_VIRT
#define ACPF_ZB_VIRT 4
#endif
constexpr int kZbVirt = ACPF_ZB_VIRT;
#ifndef ACPF_ZB_BUF
#define ACPF_ZB_BUF 2
#endif
constexpr int kZbBuf = ACPF_ZB_BUF;  // Z stage buffers (TMA ring; 4 x half-K stages measured 2% slower)

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

template <int CL>
__device__ __forceinline__ uint32_t cluster_rank() {
  if (CL == 1) return 0;
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}

// cluster-wide barrier with release/acquire semantics (orders the global v
// writes of one CTA before the other CTAs' next injection reads)
template <int CL>
__device__ __forceinline__ void cluster_sync_all() {
  if (CL == 1) {
    __syncthreads();
    return;
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// a double in CTA `rank`'s shared memory at the address of `p` in this CTA
__device__ __forceinline__ double ld_dsmem(const double* p, uint32_t rank) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(ra) : "r"(smem_u32(p)), "r"(rank));
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];\n" : "=d"(v) : "r"(ra) : "memory");
  return v;
}

// reference-style complex quotient s / v (scaled, no overflow for |v| ~ 1)
__device__ __forceinline__ double2 cdiv(double2 s, double2 v) {
  if (fabs(v.x) >= fabs(v.y)) {
    const double r = v.y / v.x, den = v.x + v.y * r;
    return make_double2((s.x + s.y * r) / den, (s.y - s.x * r) / den);
  }
  const double r = v.x / v.y, den = v.x * r + v.y;
  return make_double2((s.x * r + s.y) / den, (s.y * r - s.x) / den);
}

// NaN-propagating max (np.max semantics)
__device__ __forceinline__ double nanmax(double a, double b) {
  return (isnan(a) || a > b) ? a : b;
}

enum PassMode { kIterate = 0, kCert = 1, kMag0 = 2 };

template <int NT>
struct Smem {
  static constexpr int kCgWarp = NT / (8 * kColWarps);   // column groups per warp
};

template <int NT>
__device__ __forceinline__ int ifrag_index(int k, int col) {
  // B fragment (k x col), layout [kstep][cg][comp][lane], lane = (col%8)*4 + k%4
  return (((k >> 2) * (NT / 8) + (col >> 3)) * 2) * 32 + ((col & 7) << 2) + (k & 3);
}

struct ZbTileState {
  double* colsum;  // [NT]
  double* red;     // [kRowWarps][NT]
  int* run;        // [NT] 1 = running (writes allowed in an iterate pass)
  int* cert;       // [NT] 1 = needs the certificate pass
  double* part;    // [kZbVirt][NT] per-class column partials of a pass
};

// One sweep over all Z stages for the current tile.
template <int NT, int MODE, int CL>
__device__ void zb_pass(const ZbDeviceModel& m, const ZbBatchIO& io, int64_t tile_col0,
                        double* zs, const double* isf, uint64_t* bars, uint32_t& phase_bits,
                        ZbTileState st, int crank) {
  constexpr int CGW = Smem<NT>::kCgWarp;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rp = warp % kRowWarps, ch = warp / kRowWarps;
  const int ksteps = m.kpad >> 2;
  const int n_kc = (ksteps + kMaxKsPerStage - 1) / kMaxKsPerStage;
  // this CTA's row-block classes: its rank's (cluster of kZbVirt) or all of
  // them in order (one CTA per tile); class c = row blocks c, c + V, ...
  const int c_begin = CL == 1 ? 0 : crank, c_end = CL == 1 ? kZbVirt : crank + 1;
  auto nrb = [&](int c) { return m.n_rb > c ? (m.n_rb - c + kZbVirt - 1) / kZbVirt : 0; };
  int n_stage = 0;
  for (int c = c_begin; c < c_end; ++c) n_stage += nrb(c) * n_kc;
  // stage -> (class, row block, k chunk)
  auto decode = [&](int sidx, int& cls, int& rb, int& kc) {
    int c = c_begin, base = 0;
    while (base + nrb(c) * n_kc <= sidx) base += nrb(c++) * n_kc;
    cls = c;
    rb = c + kZbVirt * ((sidx - base) / n_kc);
    kc = (sidx - base) % n_kc;
  };
  const int stage_doubles = (ksteps < kMaxKsPerStage ? ksteps : kMaxKsPerStage) * 512;

  // Each stage is two row halves (rows 0-31 / 32-63 of the row block), each
  // a contiguous fragment block streamed by its own bulk copy onto its own
  // full barrier and released through its own empty barrier by the 16 warps
  // that read it; a leader thread per half refills it. The two halves of the
  // CTA thus only share I_l (constant during a pass) and drift independently.
  constexpr int kHalfRW = kRowWarps / 2;        // row warps per half
  const int half = rp / kHalfRW;
  const bool leader = (rp % kHalfRW) == 0 && ch == 0 && lane == 0;
  const int half_doubles = stage_doubles / 2;
  uint64_t* const fullb = bars + half * kZbBuf;                // [kZbBuf] of this half
  uint64_t* const emptyb = bars + 2 * kZbBuf + half * kZbBuf;  // [kZbBuf] of this half
  auto issue = [&](int sidx) {
    int cls_, rb, kc;
    decode(sidx, cls_, rb, kc);
    const int ks0 = kc * kMaxKsPerStage;
    const int nks = min(kMaxKsPerStage, ksteps - ks0);
    const double* src = m.zfrag + (((size_t)rb * 2 + half) * ksteps + ks0) * 256;
    const uint32_t bytes = (uint32_t)nks * 256 * 8;
    double* dst = zs + (sidx % kZbBuf) * stage_doubles + half * half_doubles;
    uint64_t* bar = fullb + (sidx % kZbBuf);
    mbar_expect_tx(bar, bytes);
    for (uint32_t off = 0; off < bytes; off += 32768u) {
      const uint32_t chunk = min(32768u, bytes - off);
      bulk_g2s(reinterpret_cast<char*>(dst) + off, reinterpret_cast<const char*>(src) + off, chunk,
               bar);
    }
  };

  // full barriers: TMA transaction count; empty barriers: one arrive per warp
  // of the half once its DMMAs on the stage are issued and complete. Parities:
  // full in bits 0..kZbBuf-1, empty (leaders only) in bits kZbBuf.. of
  // phase_bits.
  if (leader) {
    // the stage buffers may have been generic-proxy scratch since the last
    // pass (zb_injection_cta): order those accesses before the bulk writes
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    for (int k = 0; k < kZbBuf && k < n_stage; ++k) issue(k);
  }

#ifndef ACPF_ZB_4M
  // 3-multiply complex product (default; -DACPF_ZB_4M restores the 4-multiply
  // form): P1 = Zr (Ir + Ii), P2 = (Zr + Zi) Ii, P3 = (Zi - Zr) Ir;
  // Re = P1 - P2, Im = P1 + P3 — 3 DMMAs per complex k-step instead of 4, the
  // operand sums formed in registers from the same fragments (1.74M -> 1.90M
  // EULV scenarios/s on 262,144)
  double c1[kRowGroups][CGW][2], c2[kRowGroups][CGW][2], c3[kRowGroups][CGW][2];
#else
  double cr[kRowGroups][CGW][2], ci[kRowGroups][CGW][2];
#endif
  // per-lane running column partials over all row blocks (rows lane/4 of the
  // warp's two row groups); reduced across lanes/warps once per pass
  double acc[CGW][2];
#pragma unroll
  for (int b = 0; b < CGW; ++b) acc[b][0] = acc[b][1] = 0.0;
  // per-pass column reduction of the lane partials of one class: 8 row lanes
  // (fixed butterfly), then the kRowWarps row warps in fixed order
  // (the lane butterfly here, per warp; the row warps at the end of the pass)
  auto flush = [&](int cls) {
#pragma unroll
    for (int b = 0; b < CGW; ++b)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        double x = acc[b][j];
#pragma unroll
        for (int off = 4; off < 32; off <<= 1) {
          const double o = __shfl_xor_sync(0xffffffffu, x, off);
          x = (MODE == kCert) ? nanmax(x, o) : x + o;
        }
        if (lane < 4) st.red[(cls * kRowWarps + rp) * NT + (ch * CGW + b) * 8 + 2 * lane + j] = x;
        acc[b][j] = 0.0;
      }
  };
  for (int sidx = 0; sidx < n_stage; ++sidx) {
    int cls, rb, kc;
    decode(sidx, cls, rb, kc);
    const int buf = sidx % kZbBuf;
    if (kc == 0) {
#pragma unroll
      for (int a = 0; a < kRowGroups; ++a)
#pragma unroll
        for (int b = 0; b < CGW; ++b) {
#ifndef ACPF_ZB_4M
          c1[a][b][0] = c1[a][b][1] = c2[a][b][0] = c2[a][b][1] = c3[a][b][0] = c3[a][b][1] = 0.0;
#else
          cr[a][b][0] = cr[a][b][1] = ci[a][b][0] = ci[a][b][1] = 0.0;
#endif
        }
    }
    mbar_wait(fullb + buf, (phase_bits >> buf) & 1u);
    phase_bits ^= (1u << buf);
    const double* zb = zs + buf * stage_doubles + half * half_doubles;
    const int ks0 = kc * kMaxKsPerStage;
    const int nks = min(kMaxKsPerStage, ksteps - ks0);
    for (int ks = 0; ks < nks; ++ks) {
      double ar[kRowGroups], ai[kRowGroups], br[CGW], bi[CGW];
#pragma unroll
      for (int a = 0; a < kRowGroups; ++a) {
        const int rg = (rp % kHalfRW) * kRowGroups + a;  // row group within the half
        ar[a] = zb[((ks * 4 + rg) * 2 + 0) * 32 + lane];
        ai[a] = zb[((ks * 4 + rg) * 2 + 1) * 32 + lane];
      }
#pragma unroll
      for (int b = 0; b < CGW; ++b) {
        const int cg = ch * CGW + b;
        br[b] = isf[(((ks0 + ks) * (NT / 8) + cg) * 2 + 0) * 32 + lane];
        bi[b] = isf[(((ks0 + ks) * (NT / 8) + cg) * 2 + 1) * 32 + lane];
      }
#ifndef ACPF_ZB_4M
      double bs[CGW];
#pragma unroll
      for (int b = 0; b < CGW; ++b) bs[b] = br[b] + bi[b];
#pragma unroll
      for (int a = 0; a < kRowGroups; ++a) {
        const double zs_ = ar[a] + ai[a], zd = ai[a] - ar[a];
#pragma unroll
        for (int b = 0; b < CGW; ++b) {
          dmma(c1[a][b][0], c1[a][b][1], ar[a], bs[b]);
          dmma(c2[a][b][0], c2[a][b][1], zs_, bi[b]);
          dmma(c3[a][b][0], c3[a][b][1], zd, br[b]);
        }
      }
#else
#pragma unroll
      for (int a = 0; a < kRowGroups; ++a) {
        const double nai = -ai[a];
#pragma unroll
        for (int b = 0; b < CGW; ++b) {
          dmma(cr[a][b][0], cr[a][b][1], ar[a], br[b]);
          dmma(cr[a][b][0], cr[a][b][1], nai, bi[b]);
          dmma(ci[a][b][0], ci[a][b][1], ar[a], bi[b]);
          dmma(ci[a][b][0], ci[a][b][1], ai[a], br[b]);
        }
      }
#endif
    }
    // release the stage buffer (all lanes' shared reads of zb are done)
    __syncwarp();
    if (lane == 0) mbar_arrive(emptyb + buf);
    if (leader && sidx + kZbBuf < n_stage) {
      mbar_wait(emptyb + buf, (phase_bits >> (kZbBuf + buf)) & 1u);
      phase_bits ^= (1u << (kZbBuf + buf));
      issue(sidx + kZbBuf);
    }
    if (kc == n_kc - 1) {
      // ---- epilogue for row block rb (no CTA-wide synchronisation)
#pragma unroll
      for (int a = 0; a < kRowGroups; ++a) {
        const int row = rb * kZbRows + (rp * kRowGroups + a) * 8 + (lane >> 2);
        const double2 v0 = m.v0[row];
        const bool in = row < m.n;
#pragma unroll
        for (int b = 0; b < CGW; ++b) {
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int col = (ch * CGW + b) * 8 + 2 * (lane & 3) + j;
#ifndef ACPF_ZB_4M
            const double vr = (c1[a][b][j] - c2[a][b][j]) + v0.x, vi = (c1[a][b][j] + c3[a][b][j]) + v0.y;
#else
            const double vr = cr[a][b][j] + v0.x, vi = ci[a][b][j] + v0.y;
#endif
            double contrib = 0.0;
            if (MODE == kIterate) {
              if (in) {
                contrib = sqrt(vr * vr + vi * vi);
                ACPF_CHECK(!st.run[col] || (tile_col0 + col < io.batch && row < m.n));
                if (st.run[col]) io.v_out[(tile_col0 + col) * m.n + row] = make_double2(vr, vi);
              }
              acc[b][j] = acc[b][j] + contrib;
            } else if (MODE == kMag0) {
              if (in) contrib = sqrt(vr * vr + vi * vi);
              acc[b][j] = acc[b][j] + contrib;
            } else {  // certificate: |v_final - (Z i(v_final) + v0)|
              if (in && st.cert[col]) {
                ACPF_CHECK(tile_col0 + col < io.batch && row < m.n);
                const double2 vf = io.v_out[(tile_col0 + col) * m.n + row];
                const double dr = vf.x - vr, di = vf.y - vi;
                contrib = sqrt(dr * dr + di * di);
              }
              acc[b][j] = nanmax(acc[b][j], contrib);
            }
          }
        }
      }
    }
    if (kc == n_kc - 1 && rb + kZbVirt >= m.n_rb) flush(cls);  // the class's last row block
  }
  // the empty-barrier phases of the stages whose refill was not needed
  // (the last kZbBuf) still advance: keep thread 0's parity bits in sync
  if (leader) {
    for (int sidx = (n_stage > kZbBuf ? n_stage - kZbBuf : 0); sidx < n_stage; ++sidx) {
      const int buf = sidx % kZbBuf;
      mbar_wait(emptyb + buf, (phase_bits >> (kZbBuf + buf)) & 1u);
      phase_bits ^= (1u << (kZbBuf + buf));
    }
  }
  // per class: the kRowWarps row warps in fixed order (classes without row
  // blocks contribute 0); then this CTA's column sums: the classes in order
  // (one CTA per tile) or its own class (cluster)
  __syncthreads();
  if (tid < NT) {
    for (int c = c_begin; c < c_end; ++c) {
      double x = 0.0;
      if (nrb(c) > 0) {
        const double* r = st.red + (size_t)c * kRowWarps * NT;
        x = r[tid];
#pragma unroll
        for (int w = 1; w < kRowWarps; ++w) x = (MODE == kCert) ? nanmax(x, r[w * NT + tid]) : x + r[w * NT + tid];
      }
      st.part[c * NT + tid] = x;
    }
    double x = st.part[c_begin * NT + tid];
    for (int c = c_begin + 1; c < c_end; ++c)
      x = (MODE == kCert) ? nanmax(x, st.part[c * NT + tid]) : x + st.part[c * NT + tid];
    st.colsum[tid] = x;
  }
  __syncthreads();
}

// Column-owner work: build I_l for column `col` from v at the load rows.
// Returns floor slot (>= 0) on a voltage-floor violation, else -1.
template <int NT>
__device__ int zb_injection(const ZbDeviceModel& m, const ZbBatchIO& io, int64_t scen, int col,
                            bool from_v0, double* isf) {
  for (int k = 0; k < m.kpad; ++k) {
    isf[ifrag_index<NT>(k, col) + 0] = 0.0;
    isf[ifrag_index<NT>(k, col) + 32] = 0.0;
  }
  auto vat = [&](int lcol) -> double2 {
    const int row = m.l_row[lcol];
    return from_v0 ? m.v0[row] : __ldcg(io.v_out + scen * m.n + row);
  };
  // floor checks in the reference order (distribution.py:583-606)
  for (int k = 0; k < m.n_wye; ++k) {
    const double2 v = vat(m.wye_l[k]);
    if (hypot(v.x, v.y) <= m.floor) return k;
  }
  for (int k = 0; k < m.n_delta; ++k) {
    const double2 v = vat(m.dp_l[k]);
    if (hypot(v.x, v.y) <= m.floor) return m.n_wye + k;
  }
  for (int k = 0; k < m.n_delta; ++k) {
    const double2 v = vat(m.dq_l[k]);
    if (hypot(v.x, v.y) <= m.floor) return m.n_wye + m.n_delta + k;
  }
  for (int k = 0; k < m.n_delta; ++k) {
    const double2 vp = vat(m.dp_l[k]), vq = vat(m.dq_l[k]);
    if (hypot(vp.x - vq.x, vp.y - vq.y) <= m.floor) return m.n_wye + 2 * m.n_delta + k;
  }
  // wye: i[p] += -conj(s / v_p), in load order (np.add.at)
  for (int k = 0; k < m.n_wye; ++k) {
    const int lc = m.wye_l[k];
    const double2 q = cdiv(io.s_wye[scen * m.n_wye + k], vat(lc));
    const int idx = ifrag_index<NT>(lc, col);
    isf[idx] = isf[idx] + (-q.x);
    isf[idx + 32] = isf[idx + 32] + q.y;
  }
  // delta: i_line = conj(s / (v_p - v_q)); i[p] -= i_line (all k), then i[q] += i_line
  for (int pass = 0; pass < 2; ++pass) {
    for (int k = 0; k < m.n_delta; ++k) {
      const double2 vp = vat(m.dp_l[k]), vq = vat(m.dq_l[k]);
      const double2 q = cdiv(io.s_delta[scen * m.n_delta + k], make_double2(vp.x - vq.x, vp.y - vq.y));
      const int lc = pass == 0 ? m.dp_l[k] : m.dq_l[k];
      const int idx = ifrag_index<NT>(lc, col);
      if (pass == 0) {
        isf[idx] = isf[idx] + (-q.x);
        isf[idx + 32] = isf[idx + 32] + q.y;
      } else {
        isf[idx] = isf[idx] + q.x;
        isf[idx + 32] = isf[idx + 32] + (-q.y);
      }
    }
  }
  return -1;
}

// Whole-CTA version of zb_injection for the columns with want[col] set (used
// when its scratch fits the Z stage buffers, which are idle between passes):
//   1. all threads gather v at the load rows of every wanted column into
//      scratch (independent loads: one latency round instead of one per load),
//   2. all threads compute the per-load currents (and the voltage-floor
//      checks, first violation in the reference order via atomicMin),
//   3. the column owner accumulates them into I_l in the reference order.
// The currents are the same cdiv() values added in the same order as
// zb_injection, so I_l is bitwise identical. fslot[col] gets the floor slot or -1.
template <int NT>
__device__ void zb_injection_cta(const ZbDeviceModel& m, const ZbBatchIO& io, int64_t col0, const int* want,
                                 bool from_v0, double* isf, double2* scratch, int* fslot) {
  const int tid = threadIdx.x;
  const int nl = m.n_l, nld = m.n_wye + m.n_delta;
  double2* vl = scratch;                  // [NT][n_l]
  double2* qb = scratch + (size_t)NT * nl;  // [NT][n_wye + n_delta]
  if (tid < NT) fslot[tid] = 0x7fffffff;
  for (int idx = tid; idx < NT * nl; idx += kThreads) {
    const int col = idx / nl, lc = idx - col * nl;
    if (!want[col]) continue;
    const int row = m.l_row[lc];
    vl[idx] = from_v0 ? m.v0[row] : __ldcg(io.v_out + (col0 + col) * m.n + row);
  }
  __syncthreads();
  for (int idx = tid; idx < NT * nld; idx += kThreads) {
    const int col = idx / nld, k = idx - col * nld;
    if (!want[col]) continue;
    const int64_t scen = col0 + col;
    const double2* v = vl + (size_t)col * nl;
    double2 q;
    int slot = 0x7fffffff;
    if (k < m.n_wye) {
      const double2 vp = v[m.wye_l[k]];
      if (hypot(vp.x, vp.y) <= m.floor) slot = k;
      q = cdiv(io.s_wye[scen * m.n_wye + k], vp);
    } else {
      const int d = k - m.n_wye;
      const double2 vp = v[m.dp_l[d]], vq = v[m.dq_l[d]];
      if (hypot(vp.x, vp.y) <= m.floor) slot = m.n_wye + d;
      else if (hypot(vq.x, vq.y) <= m.floor) slot = m.n_wye + m.n_delta + d;
      else if (hypot(vp.x - vq.x, vp.y - vq.y) <= m.floor) slot = m.n_wye + 2 * m.n_delta + d;
      q = cdiv(io.s_delta[scen * m.n_delta + d], make_double2(vp.x - vq.x, vp.y - vq.y));
    }
    qb[idx] = q;
    if (slot != 0x7fffffff) atomicMin(fslot + col, slot);
  }
  __syncthreads();
  if (tid < NT && want[tid]) {
    const int col = tid;
    if (fslot[col] == 0x7fffffff) {
      fslot[col] = -1;
      for (int k = 0; k < m.kpad; ++k) {
        isf[ifrag_index<NT>(k, col) + 0] = 0.0;
        isf[ifrag_index<NT>(k, col) + 32] = 0.0;
      }
      const double2* q = qb + (size_t)col * nld;
      for (int k = 0; k < m.n_wye; ++k) {  // wye: i[p] += -conj(s / v_p)
        const int idx = ifrag_index<NT>(m.wye_l[k], col);
        isf[idx] = isf[idx] + (-q[k].x);
        isf[idx + 32] = isf[idx + 32] + q[k].y;
      }
      for (int k = 0; k < m.n_delta; ++k) {  // delta: i[p] -= i_line (all k) ...
        const int idx = ifrag_index<NT>(m.dp_l[k], col);
        isf[idx] = isf[idx] + (-q[m.n_wye + k].x);
        isf[idx + 32] = isf[idx + 32] + q[m.n_wye + k].y;
      }
      for (int k = 0; k < m.n_delta; ++k) {  // ... then i[q] += i_line
        const int idx = ifrag_index<NT>(m.dq_l[k], col);
        isf[idx] = isf[idx] + q[m.n_wye + k].x;
        isf[idx + 32] = isf[idx + 32] + (-q[m.n_wye + k].y);
      }
    }
  }
}

// Combine the cluster's per-CTA column partials (sum, or NaN-propagating max
// for the certificate) in rank order; every CTA ends with the same totals.
template <int NT, int CL, bool MAX>
__device__ __forceinline__ void zb_cluster_combine(double* colsum) {
  if (CL == 1) return;      // colsum already holds the totals
  cluster_sync_all<CL>();   // every CTA's partial is in its colsum
  const int tid = threadIdx.x;
  double x = 0.0;
  if (tid < NT) {
    x = ld_dsmem(colsum + tid, 0);
#pragma unroll
    for (int r = 1; r < CL; ++r) {
      const double y = ld_dsmem(colsum + tid, (uint32_t)r);
      x = MAX ? nanmax(x, y) : x + y;
    }
  }
  cluster_sync_all<CL>();  // all remote reads done before colsum is overwritten
  if (tid < NT) colsum[tid] = x;
  __syncthreads();
}

template <int NT, int CL>
__global__ void __launch_bounds__(kThreads, ACPF_ZB_MINB)
    zbus_kernel(ZbDeviceModel m, ZbBatchIO io, double tol, int max_iter, int mag0_mode,
                double* mag0_out) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int ksteps = m.kpad >> 2;
  const int stage_doubles = (ksteps < kMaxKsPerStage ? ksteps : kMaxKsPerStage) * 512;
  double* zs = reinterpret_cast<double*>(smem_raw);
  double* isf = zs + kZbBuf * stage_doubles;
  double* colsum = isf + (size_t)ksteps * NT * 8;
  double* red = colsum + NT;
  double* mag = red + kZbVirt * kRowWarps * NT;
  double* delta = mag + NT;
  double* resid = delta + NT;
  int* run = reinterpret_cast<int*>(resid + NT);
  int* cert = run + NT;
  int* stat = cert + NT;
  int* iters = stat + NT;
  int* fslot = iters + NT;
  uint64_t* bars = reinterpret_cast<uint64_t*>(fslot + NT + (NT & 1));
  double* part = reinterpret_cast<double*>(bars + 4 * kZbBuf);  // [kZbVirt][NT]

  const int tid = threadIdx.x;
  const int crank = (int)cluster_rank<CL>();
  if (tid == 0) {
    for (int b = 0; b < 2 * kZbBuf; ++b) {
      mbar_init(bars + b, 1);                              // half-stage full (TMA transaction count)
      mbar_init(bars + 2 * kZbBuf + b, kThreads / 64);     // half-stage empty (one arrive per warp of the half)
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  uint32_t phase_bits = 0;
  ZbTileState st{colsum, red, run, cert, part};
  // the CTA-wide injection needs [NT][n_l] voltages + [NT][loads] currents of
  // scratch in the (then idle) Z stage buffers
  const bool par_inj = (size_t)NT * (m.n_l + m.n_wye + m.n_delta) * 2 <= kZbBuf * (size_t)stage_doubles;

  if (mag0_mode) {
    for (int k = tid; k < ksteps * NT * 8; k += kThreads) isf[k] = 0.0;
    if (tid < NT) colsum[tid] = 0.0, run[tid] = 0;
    __syncthreads();
    zb_pass<NT, kMag0, CL>(m, io, 0, zs, isf, bars, phase_bits, st, crank);
    zb_cluster_combine<NT, CL, false>(colsum);
    if (tid == 0 && crank == 0) *mag0_out = colsum[0];
    return;
  }

  const int64_t n_tiles = (io.batch + NT - 1) / NT;
  const int cid = blockIdx.x / CL, ncl = gridDim.x / CL;
  for (int64_t tile = cid; tile < n_tiles; tile += ncl) {
    const int64_t col0 = tile * NT;
    const int64_t scen = col0 + tid;
    if (tid < NT) {
      const bool live = scen < io.batch;
      run[tid] = live;
      cert[tid] = 0;
      stat[tid] = live ? -1 : -2;
      mag[tid] = m.mag0;
      delta[tid] = __longlong_as_double(0x7ff0000000000000LL);
      resid[tid] = 0.0;
      iters[tid] = 0;
      fslot[tid] = -1;
    }
    // ---- sweeps
    for (int k = 1; k <= max_iter; ++k) {
      int* const inj_slot = reinterpret_cast<int*>(red);  // red is free between passes
      if (par_inj) {
        __syncthreads();  // run[] of the previous sweep visible to every thread
        zb_injection_cta<NT>(m, io, col0, run, k == 1, isf, reinterpret_cast<double2*>(zs), inj_slot);
      }
      if (tid < NT) {
        if (run[tid]) {
          const int fs = par_inj ? inj_slot[tid] : zb_injection<NT>(m, io, scen, tid, k == 1, isf);
          if (fs >= 0) {
            run[tid] = 0;
            stat[tid] = ACPF_ZB_FLOOR;
            iters[tid] = k;
            fslot[tid] = fs;
            resid[tid] = __longlong_as_double(0x7ff0000000000000LL);
            if (k == 1 && crank == 0)
              for (int r = 0; r < m.n; ++r) io.v_out[scen * m.n + r] = m.v0[r];
          }
        }
        if (!run[tid])
          for (int q = 0; q < m.kpad; ++q) {
            isf[ifrag_index<NT>(q, tid)] = 0.0;
            isf[ifrag_index<NT>(q, tid) + 32] = 0.0;
          }
        colsum[tid] = 0.0;
      }
      const int any = __syncthreads_or(tid < NT && run[tid]);
      if (!any) break;
      zb_pass<NT, kIterate, CL>(m, io, col0, zs, isf, bars, phase_bits, st, crank);
      zb_cluster_combine<NT, CL, false>(colsum);
      if (tid < NT && run[tid]) {
        const double s = colsum[tid];
        const double d = fabs(s - mag[tid]);
        mag[tid] = s;
        delta[tid] = d;
        if (d <= tol) {
          run[tid] = 0;
          stat[tid] = ACPF_ZB_CONVERGED;
          iters[tid] = k;
        } else if (k == max_iter) {
          run[tid] = 0;
          stat[tid] = ACPF_ZB_MAX_ITER;
          iters[tid] = k;
        }
      }
      __syncthreads();
    }
    // ---- certificate ||v - (Z i(v) + v0)||inf
    if (par_inj) {
      int* const inj_slot = reinterpret_cast<int*>(red);
      if (tid < NT) cert[tid] = stat[tid] == ACPF_ZB_CONVERGED || stat[tid] == ACPF_ZB_MAX_ITER;
      __syncthreads();
      zb_injection_cta<NT>(m, io, col0, cert, false, isf, reinterpret_cast<double2*>(zs), inj_slot);
    }
    if (tid < NT) {
      const bool want = stat[tid] == ACPF_ZB_CONVERGED || stat[tid] == ACPF_ZB_MAX_ITER;
      cert[tid] = 0;
      colsum[tid] = 0.0;
      if (want) {
        const int fs = par_inj ? reinterpret_cast<int*>(red)[tid] : zb_injection<NT>(m, io, scen, tid, false, isf);
        if (fs >= 0) {
          resid[tid] = __longlong_as_double(0x7ff0000000000000LL);
        } else {
          cert[tid] = 1;
        }
      }
      if (!cert[tid])
        for (int q = 0; q < m.kpad; ++q) {
          isf[ifrag_index<NT>(q, tid)] = 0.0;
          isf[ifrag_index<NT>(q, tid) + 32] = 0.0;
        }
    }
    const int anyc = __syncthreads_or(tid < NT && cert[tid]);
    if (anyc) {
      zb_pass<NT, kCert, CL>(m, io, col0, zs, isf, bars, phase_bits, st, crank);
      zb_cluster_combine<NT, CL, true>(colsum);
      if (tid < NT && cert[tid]) resid[tid] = colsum[tid];
    }
    if (tid < NT && scen < io.batch && crank == 0) {
      if (io.converged) io.converged[scen] = stat[tid] == ACPF_ZB_CONVERGED;
      if (io.iterations) io.iterations[scen] = iters[tid];
      if (io.final_delta) io.final_delta[scen] = delta[tid];
      if (io.residual) io.residual[scen] = resid[tid];
      if (io.status) io.status[scen] = stat[tid];
      if (io.floor_slot) io.floor_slot[scen] = fslot[tid];
    }
    __syncthreads();
  }
}

template <int NT>
size_t zbus_smem_bytes(int kpad) {
  const int ksteps = kpad >> 2;
  const int stage_doubles = (ksteps < kMaxKsPerStage ? ksteps : kMaxKsPerStage) * 512;
  size_t d = kZbBuf * (size_t)stage_doubles + (size_t)ksteps * NT * 8 + NT + kZbVirt * kRowWarps * NT + 3 * NT;
  size_t bytes = d * 8 + (5 * NT + 2) * 4 + 32 * kZbBuf + 16;
  return bytes + (size_t)kZbVirt * NT * 8;  // per-class partials (after the barriers)
}

template <int NT, int CL>
cudaError_t launch_ntc(const ZbDeviceModel& m, const ZbBatchIO& io, double tol, int max_iter, bool mag0_mode,
                       double* mag0_out, cudaStream_t stream, int clusters, size_t smem) {
  if (CL == 1) {
    zbus_kernel<NT, 1><<<clusters, kThreads, smem, stream>>>(m, io, tol, max_iter, mag0_mode ? 1 : 0, mag0_out);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.gridDim = dim3((unsigned)(clusters * CL), 1, 1);
  return cudaLaunchKernelEx(&cfg, zbus_kernel<NT, CL>, m, io, tol, max_iter, mag0_mode ? 1 : 0, mag0_out);
}

// clusters of CL CTAs that can be resident at once (clusters live inside a GPC)
template <int NT, int CL>
int resident_clusters(size_t smem, int sms) {
  // cached per (device, shared memory of the feeder); plans on several
  // devices are driven from concurrent host threads
  static std::mutex mu;
  static std::map<std::pair<int, size_t>, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> lk(mu);
    const auto it = cache.find({dev, smem});
    if (it != cache.end()) return it->second;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.gridDim = dim3((unsigned)(sms / CL * CL), 1, 1);
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, zbus_kernel<NT, CL>, &cfg) != cudaSuccess || n <= 0) {
    cudaGetLastError();
    n = 0;  // no cluster launch possible: one CTA per tile
  }
  std::lock_guard<std::mutex> lk(mu);
  cache[{dev, smem}] = n;
  return n;
}

template <int NT>
cudaError_t launch_nt(const ZbDeviceModel& m, const ZbBatchIO& io, double tol, int max_iter,
                      bool mag0_mode, double* mag0_out, cudaStream_t stream) {
  const size_t smem = zbus_smem_bytes<NT>(m.kpad);
  cudaError_t err = cudaFuncSetAttribute(zbus_kernel<NT, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
  if (err == cudaSuccess)
    err = cudaFuncSetAttribute(zbus_kernel<NT, kZbVirt>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err == cudaSuccess)
    err = cudaFuncSetAttribute(zbus_kernel<NT, kZbVirt>, cudaFuncAttributeNonPortableClusterSizeAllowed, 0);
  if (err != cudaSuccess) return err;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t tiles = mag0_mode ? 1 : (io.batch + NT - 1) / NT;
  // small batches: one cluster per tile (ACPF_ZB_CLUSTER=0 disables);
  // otherwise one CTA per tile (same bits)
  static const bool allow = [] {
    const char* v = std::getenv("ACPF_ZB_CLUSTER");
    return !(v && v[0] == '0');
  }();
  // (only when every CTA of the cluster has row blocks to stream)
  const int rc = (allow && !mag0_mode && kZbVirt > 1 && m.n_rb >= 2 * kZbVirt)
                     ? resident_clusters<NT, kZbVirt>(smem, sms) : 0;
  // a tile takes ~1/kZbVirt of the time on a cluster: worth it while the
  // tiles fit in up to kZbVirt - 1 waves of clusters
  if (rc > 0 && tiles <= (int64_t)(kZbVirt - 1) * rc)
    return launch_ntc<NT, kZbVirt>(m, io, tol, max_iter, mag0_mode, mag0_out, stream,
                                   (int)(tiles < rc ? tiles : rc), smem);
  const int64_t slots = (int64_t)sms * ACPF_ZB_MINB;
  const int grid = (int)(tiles < slots ? tiles : slots);
  return launch_ntc<NT, 1>(m, io, tol, max_iter, mag0_mode, mag0_out, stream, grid, smem);
}

}  // namespace

size_t zbus_frag_doubles(int n_rb, int kpad) { return (size_t)n_rb * (kpad >> 2) * 512; }

// Host: pack Z[:, l] ([n][n_l] interleaved complex) into DMMA A-fragment
// order: [row block][row half][kstep][row group 0..3][re|im][lane], lane t
// holds Z[rb*64 + (4*half + rg)*8 + t/4][ks*4 + t%4] (zero padded); each row
// half of a stage is one contiguous bulk copy.
void zbus_pack_fragments(const double* zl, int n, int n_l, int n_rb, int kpad, double* out) {
  const int ksteps = kpad >> 2;
  size_t o = 0;
  for (int rb = 0; rb < n_rb; ++rb)
    for (int half = 0; half < 2; ++half)
    for (int ks = 0; ks < ksteps; ++ks)
      for (int rg = 0; rg < 4; ++rg)
        for (int comp = 0; comp < 2; ++comp)
          for (int t = 0; t < 32; ++t) {
            const int row = rb * kZbRows + (4 * half + rg) * 8 + (t >> 2);
            const int k = ks * 4 + (t & 3);
            out[o++] = (row < n && k < n_l) ? zl[((size_t)row * n_l + k) * 2 + comp] : 0.0;
          }
}

cudaError_t launch_zbus(const ZbDeviceModel& m, const ZbBatchIO& io, double tol, int max_iter,
                        bool mag0_mode, double* mag0_out, int* launches, cudaStream_t stream) {
  if (launches) *launches = 1;
  // 64-scenario tiles unless that leaves SMs idle (small batches) or the load
  // columns need the 32-wide tile's smaller I_l; per-column reduction orders
  // do not depend on the tile width, so both give the same bits
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const bool small = !mag0_mode && (io.batch + 63) / 64 < sms;
  // ACPF_ZB_NT64=1: 64-wide tiles for large batches (the round-1 shape, with
  // 32 warps: ACPF_ZB_COL_WARPS=4); 32-wide tiles on 16 warps measured faster
  // at every batch size (122 registers, no spills; 64-wide at 16 warps spills)
  static const bool nt64 = [] {
    const char* v = std::getenv("ACPF_ZB_NT64");
    return v && v[0] == '1';
  }();
  if (nt64 && m.kpad <= 64 && !small) return launch_nt<64>(m, io, tol, max_iter, mag0_mode, mag0_out, stream);
  return launch_nt<32>(m, io, tol, max_iter, mag0_mode, mag0_out, stream);
}

}  // namespace acpf
