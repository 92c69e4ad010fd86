// Seeded scenario inputs generated on the device.
//
// Bitwise replica of the reference generator (batch.py:45-60): scenario i's
// multipliers are the first n doubles of numpy's Generator(Philox(key=[seed, i])),
// i.e. Philox4x64-10 with key (seed, i) and counter values 1, 2, ... (numpy
// increments the counter before each block), each 64-bit output x mapped to
// u = (x >> 11) * 2^-53, and m = (1 - spread) + (2 spread) * u. The load
// scaling follows batch.py:121-151 with every multiply/subtract rounded
// separately (no FMA contraction), so the device inputs are bit-identical to
// make_scenario_arrays on the host.

#include "acpf_internal.cuh"

namespace acpf {

namespace {

struct U4 {
  uint64_t x, y, z, w;
};

__device__ __forceinline__ void mulhilo64(uint64_t a, uint64_t b, uint64_t& hi, uint64_t& lo) {
  lo = a * b;
  hi = __umul64hi(a, b);
}

// Random123 Philox4x64 with 10 rounds (the numpy bit generator)
__device__ __forceinline__ U4 philox4x64_10(U4 ctr, uint64_t k0, uint64_t k1) {
  const uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
  const uint64_t W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += W0;
      k1 += W1;
    }
    uint64_t hi0, lo0, hi1, lo1;
    mulhilo64(M0, ctr.x, hi0, lo0);
    mulhilo64(M1, ctr.z, hi1, lo1);
    ctr = U4{hi1 ^ ctr.y ^ k0, lo1, hi0 ^ ctr.w ^ k1, lo0};
  }
  return ctr;
}

// the 4 multipliers of draws 4*blk .. 4*blk+3 of scenario i
__device__ __forceinline__ void multipliers4(uint64_t seed, uint64_t i, uint64_t blk, double lo,
                                             double width, double m[4]) {
  const U4 o = philox4x64_10(U4{blk + 1, 0, 0, 0}, seed, i);
  const uint64_t v[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double u = (double)(v[k] >> 11) * (1.0 / 9007199254740992.0);
    m[k] = __dadd_rn(lo, __dmul_rn(width, u));
  }
}

__global__ void philox_multipliers_kernel(uint64_t seed, int64_t start, int64_t count, int n_elem,
                                          double lo, double width, double* out) {
  const int nblk = (n_elem + 3) / 4;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count * nblk) return;
  const int64_t row = t / nblk;
  const int blk = (int)(t % nblk);
  double m[4];
  multipliers4(seed, (uint64_t)(start + row), (uint64_t)blk, lo, width, m);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int e = blk * 4 + k;
    if (e < n_elem) out[row * n_elem + e] = m[k];
  }
}

// base rows: p_spec = p_gen - p_load (p_load is 0 off the load elements)
__global__ void nr_base_rows_kernel(int64_t count, int n_theta, int n_q, const double* p_base,
                                    const double* q_base, double* p_spec, double* q_spec) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int nj = n_theta + n_q;
  if (t >= count * nj) return;
  const int64_t row = t / nj;
  const int k = (int)(t % nj);
  if (k < n_theta)
    p_spec[row * n_theta + k] = p_base[k];
  else
    q_spec[row * n_q + (k - n_theta)] = q_base[k - n_theta];
}

// load elements: p_spec = p_gen - (p_load * m), q likewise
__global__ void nr_scale_kernel(uint64_t seed, int64_t start, int64_t count, int n_elem, double lo,
                                double width, const int32_t* elem_tpos, const int32_t* elem_qidx,
                                const double* elem_pl, const double* elem_ql, const double* elem_pg,
                                const double* elem_qg, int n_theta, int n_q, double* p_spec,
                                double* q_spec) {
  const int nblk = (n_elem + 3) / 4;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count * nblk) return;
  const int64_t row = t / nblk;
  const int blk = (int)(t % nblk);
  double m[4];
  multipliers4(seed, (uint64_t)(start + row), (uint64_t)blk, lo, width, m);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int e = blk * 4 + k;
    if (e >= n_elem) break;
    const int tp = elem_tpos[e], qi = elem_qidx[e];
    if (tp >= 0) p_spec[row * n_theta + tp] = __dsub_rn(elem_pg[e], __dmul_rn(elem_pl[e], m[k]));
    if (qi >= 0) q_spec[row * n_q + qi] = __dsub_rn(elem_qg[e], __dmul_rn(elem_ql[e], m[k]));
  }
}

// distribution: wye load w scaled by m (complex * real), delta likewise
__global__ void zb_scale_kernel(uint64_t seed, int64_t start, int64_t count, int n_elem, double lo,
                                double width, const int32_t* elem_target, const double2* wye_s,
                                const double2* delta_s, int n_wye, int n_delta, double2* s_wye,
                                double2* s_delta) {
  const int nblk = (n_elem + 3) / 4;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count * nblk) return;
  const int64_t row = t / nblk;
  const int blk = (int)(t % nblk);
  double m[4];
  multipliers4(seed, (uint64_t)(start + row), (uint64_t)blk, lo, width, m);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int e = blk * 4 + k;
    if (e >= n_elem) break;
    const int tg = elem_target[e];
    if (tg >= 0) {
      const double2 s = wye_s[tg];
      s_wye[row * n_wye + tg] = make_double2(__dmul_rn(s.x, m[k]), __dmul_rn(s.y, m[k]));
    } else {
      const int d = -tg - 1;
      const double2 s = delta_s[d];
      s_delta[row * n_delta + d] = make_double2(__dmul_rn(s.x, m[k]), __dmul_rn(s.y, m[k]));
    }
  }
}

unsigned grid_for(int64_t n, int tpb) { return (unsigned)((n + tpb - 1) / tpb); }

}  // namespace

cudaError_t launch_philox_multipliers(uint64_t seed, int64_t start, int64_t count, int n_elem,
                                      double spread, double* out, cudaStream_t st) {
  const double lo = 1.0 - spread, width = 2.0 * spread;
  const int64_t n = count * ((n_elem + 3) / 4);
  if (n > 0) philox_multipliers_kernel<<<grid_for(n, 256), 256, 0, st>>>(seed, start, count, n_elem, lo, width, out);
  return cudaGetLastError();
}

cudaError_t launch_nr_scenarios(const NrScenarioArgs& a, cudaStream_t st) {
  const double lo = 1.0 - a.spread, width = 2.0 * a.spread;
  const int64_t nb = a.count * (int64_t)(a.n_theta + a.n_q);
  if (nb > 0)
    nr_base_rows_kernel<<<grid_for(nb, 256), 256, 0, st>>>(a.count, a.n_theta, a.n_q, a.p_base, a.q_base,
                                                          a.p_spec, a.q_spec);
  const int64_t ns = a.count * ((a.n_elem + 3) / 4);
  if (ns > 0)
    nr_scale_kernel<<<grid_for(ns, 256), 256, 0, st>>>(a.seed, a.start, a.count, a.n_elem, lo, width,
                                                       a.elem_tpos, a.elem_qidx, a.elem_pl, a.elem_ql,
                                                       a.elem_pg, a.elem_qg, a.n_theta, a.n_q, a.p_spec,
                                                       a.q_spec);
  return cudaGetLastError();
}

cudaError_t launch_zb_scenarios(const ZbScenarioArgs& a, cudaStream_t st) {
  const double lo = 1.0 - a.spread, width = 2.0 * a.spread;
  const int64_t ns = a.count * ((a.n_elem + 3) / 4);
  if (ns > 0)
    zb_scale_kernel<<<grid_for(ns, 256), 256, 0, st>>>(a.seed, a.start, a.count, a.n_elem, lo, width,
                                                       a.elem_target, a.wye_s, a.delta_s, a.n_wye,
                                                       a.n_delta, a.s_wye, a.s_delta);
  return cudaGetLastError();
}

}  // namespace acpf
