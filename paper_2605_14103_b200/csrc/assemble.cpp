// Native host model build: pi-model Ybus and the
// three-phase node-phase Y, assembled in C++ and bit-identical to the
// reference's NumPy/SciPy assembly.
//
// Reference: build_ybus (network.py:450-496) and build_three_phase_ybus
// (distribution.py:356-391). Bit-identity needs two things restated exactly:
//  * the stamp arithmetic of CPython 3.12 complex numbers (a float operand is
//    promoted to x + 0j, products and Smith-style quotients as in
//    Objects/complexobject.c), so signed zeros and rounding match;
//  * SciPy's COO -> CSR canonicalisation: entries scattered into rows in
//    input order (coo_tocsr), each row sorted by column with std::sort on
//    the column key only (csr_sort_indices, the same introsort, so the order
//    of duplicates is the same), duplicates summed left to right
//    (csr_sum_duplicates), then exact 0+0j entries dropped.
// Host code only; x86-64 without -mfma, so no contraction changes a sum.

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "acpf_internal.cuh"

namespace acpf {

namespace {

struct Cx {
  double re, im;
};

inline Cx c_add(Cx a, Cx b) { return {a.re + b.re, a.im + b.im}; }
inline Cx c_neg(Cx a) { return {-a.re, -a.im}; }
inline Cx c_conj(Cx a) { return {a.re, -a.im}; }
inline Cx c_prod(Cx a, Cx b) { return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }
inline Cx c_of(double x) { return {x, 0.0}; }

// _Py_c_quot (CPython 3.12); false on division by zero (ZeroDivisionError)
inline bool c_quot(Cx a, Cx b, Cx& r) {
  const double abr = b.re < 0 ? -b.re : b.re;
  const double abi = b.im < 0 ? -b.im : b.im;
  if (abr >= abi) {
    if (abr == 0.0) return false;
    const double ratio = b.im / b.re;
    const double denom = b.re + b.im * ratio;
    r.re = (a.re + a.im * ratio) / denom;
    r.im = (a.im - a.re * ratio) / denom;
  } else if (abi >= abr) {
    const double ratio = b.re / b.im;
    const double denom = b.re * ratio + b.im;
    r.re = (a.re * ratio + a.im) / denom;
    r.im = (a.im * ratio - a.re) / denom;
  } else {
    r.re = r.im = std::nan("");
  }
  return true;
}

using Entry = std::pair<int32_t, std::complex<double>>;

bool kv_less(const Entry& a, const Entry& b) { return a.first < b.first; }

// scipy: coo_matrix((val, (row, col))).tocsr(); .sum_duplicates(); drop 0+0j
// (the reference's separate real/imaginary triplets lose exact zeros,
// network.py:487-495; eliminate_zeros for the three-phase Y)
void canonical_csr(int n, const std::vector<int32_t>& row, const std::vector<int32_t>& col,
                   const std::vector<Cx>& val, std::vector<int32_t>& rp, std::vector<int32_t>& cj,
                   std::vector<Cx>& x) {
  const size_t nnz = row.size();
  std::vector<int32_t> ptr(n + 1, 0);
  for (size_t k = 0; k < nnz; ++k) {
    if (row[k] < 0 || row[k] >= n || col[k] < 0 || col[k] >= n) throw std::invalid_argument("index out of range");
    ++ptr[row[k] + 1];
  }
  for (int i = 0; i < n; ++i) ptr[i + 1] += ptr[i];
  std::vector<Entry> ent(nnz);
  {
    std::vector<int32_t> fill(ptr.begin(), ptr.end() - 1);
    for (size_t k = 0; k < nnz; ++k) ent[fill[row[k]]++] = {col[k], {val[k].re, val[k].im}};
  }
  rp.assign(n + 1, 0);
  cj.clear();
  x.clear();
  std::vector<Entry> tmp;
  for (int i = 0; i < n; ++i) {
    tmp.assign(ent.begin() + ptr[i], ent.begin() + ptr[i + 1]);
    std::sort(tmp.begin(), tmp.end(), kv_less);
    for (size_t jj = 0; jj < tmp.size();) {
      const int32_t j = tmp[jj].first;
      double re = tmp[jj].second.real(), im = tmp[jj].second.imag();
      for (++jj; jj < tmp.size() && tmp[jj].first == j; ++jj) {
        re += tmp[jj].second.real();
        im += tmp[jj].second.imag();
      }
      if (re != 0.0 || im != 0.0 || std::isnan(re) || std::isnan(im)) {
        cj.push_back(j);
        x.push_back({re, im});
      }
    }
    rp[i + 1] = (int32_t)cj.size();
  }
}

int64_t emit(const std::vector<int32_t>& rp, const std::vector<int32_t>& cj, const std::vector<Cx>& x,
             int64_t capacity, int32_t* rowptr, int32_t* col, double* re, double* im, bool plus_zero) {
  const int64_t nnz = (int64_t)cj.size();
  if (capacity >= nnz && rowptr && (nnz == 0 || (col && re && im))) {
    std::memcpy(rowptr, rp.data(), rp.size() * sizeof(int32_t));
    for (int64_t k = 0; k < nnz; ++k) {
      col[k] = cj[k];
      // the reference rebuilds Ybus values as G + 1j B: +0.0 for a zero part
      re[k] = plus_zero ? x[k].re + 0.0 : x[k].re;
      im[k] = plus_zero ? x[k].im + 0.0 : x[k].im;
    }
  }
  return nnz;
}

}  // namespace

}  // namespace acpf

using namespace acpf;

extern "C" {

acpf_status acpf_ybus_build(int32_t n_bus, int32_t n_branch, const int32_t* from_idx, const int32_t* to_idx,
                            const double* r, const double* x, const double* b_ch, const double* tap,
                            const double* shift, const uint8_t* in_service, const double* gs, const double* bs,
                            int64_t capacity, int32_t* rowptr, int32_t* col, double* re, double* im,
                            int64_t* nnz_out) {
  if (n_bus <= 0 || n_branch < 0 || !gs || !bs || !nnz_out ||
      (n_branch && (!from_idx || !to_idx || !r || !x || !b_ch || !tap || !shift || !in_service))) {
    set_error("acpf_ybus_build: invalid argument");
    return ACPF_EINVAL;
  }
  try {
    std::vector<int32_t> rows, cols;
    std::vector<Cx> vals;
    rows.reserve(4 * (size_t)n_branch + n_bus);
    cols.reserve(rows.capacity());
    vals.reserve(rows.capacity());
    for (int32_t k = 0; k < n_branch; ++k) {
      if (!in_service[k]) continue;
      if (r[k] == 0.0 && x[k] == 0.0) {
        set_error("acpf_ybus_build: in-service branch " + std::to_string(k) + " has r = x = 0");
        return ACPF_EINVAL;
      }
      // _pi_stamps: series = 1 / (r + jx); shunt_half = 0.5j * b_ch;
      // a = tap * exp(1j * shift)
      Cx series, yff, yft, ytf;
      const Cx z{r[k], x[k]};
      if (!c_quot(c_of(1.0), z, series)) {
        set_error("acpf_ybus_build: complex division by zero");
        return ACPF_EINVAL;
      }
      const Cx shunt_half = c_prod({0.0, 0.5}, c_of(b_ch[k]));
      const Cx jd = c_prod({0.0, 1.0}, c_of(shift[k]));
      const double l = std::exp(jd.re);
      const Cx ejd{l * std::cos(jd.im), l * std::sin(jd.im)};
      const Cx a = c_prod(c_of(tap[k]), ejd);
      const Cx ss = c_add(series, shunt_half);
      if (!c_quot(ss, c_of(tap[k] * tap[k]), yff) || !c_quot(c_neg(series), c_conj(a), yft) ||
          !c_quot(c_neg(series), a, ytf)) {
        set_error("acpf_ybus_build: complex division by zero");
        return ACPF_EINVAL;
      }
      const int32_t f = from_idx[k], t = to_idx[k];
      const int32_t rr[4] = {f, t, f, t}, cc[4] = {f, t, t, f};
      const Cx vv[4] = {yff, ss, yft, ytf};
      for (int q = 0; q < 4; ++q) rows.push_back(rr[q]), cols.push_back(cc[q]), vals.push_back(vv[q]);
    }
    for (int32_t i = 0; i < n_bus; ++i)
      if (gs[i] != 0.0 || bs[i] != 0.0 || std::isnan(gs[i]) || std::isnan(bs[i]))
        rows.push_back(i), cols.push_back(i), vals.push_back({gs[i], bs[i]});
    std::vector<int32_t> rp, cj;
    std::vector<Cx> xv;
    canonical_csr(n_bus, rows, cols, vals, rp, cj, xv);
    *nnz_out = emit(rp, cj, xv, capacity, rowptr, col, re, im, true);
  } catch (const std::exception& ex) {
    set_error(std::string("acpf_ybus_build: ") + ex.what());
    return ACPF_EINVAL;
  }
  return ACPF_OK;
}

acpf_status acpf_y3_build(int32_t n, int32_t n_blocks, const int32_t* block_ptr, const int32_t* idx,
                          const double* val, int64_t capacity, int32_t* rowptr, int32_t* col, double* re,
                          double* im, int64_t* nnz_out) {
  if (n <= 0 || n_blocks < 0 || !nnz_out || (n_blocks && (!block_ptr || !idx || !val))) {
    set_error("acpf_y3_build: invalid argument");
    return ACPF_EINVAL;
  }
  try {
    // block b: square k x k, k = block_ptr[b+1] - block_ptr[b] phases; row
    // indices idx[2 p0 .. 2 p0 + k), column indices idx[2 p0 + k .. 2 p0 + 2k)
    // (p0 = block_ptr[b]); values row-major at val[2 * (sum of k^2 before)]
    std::vector<int32_t> rows, cols;
    std::vector<Cx> vals;
    size_t voff = 0;
    for (int32_t b = 0; b < n_blocks; ++b) {
      const int32_t p0 = block_ptr[b], k = block_ptr[b + 1] - p0;
      if (k < 0) throw std::invalid_argument("bad block_ptr");
      const int32_t* ri = idx + 2 * (size_t)p0;
      const int32_t* ci = ri + k;
      for (int32_t i = 0; i < k; ++i)
        for (int32_t j = 0; j < k; ++j, ++voff) {
          rows.push_back(ri[i]);
          cols.push_back(ci[j]);
          vals.push_back({val[2 * voff], val[2 * voff + 1]});
        }
    }
    std::vector<int32_t> rp, cj;
    std::vector<Cx> xv;
    canonical_csr(n, rows, cols, vals, rp, cj, xv);
    *nnz_out = emit(rp, cj, xv, capacity, rowptr, col, re, im, false);
  } catch (const std::exception& ex) {
    set_error(std::string("acpf_y3_build: ") + ex.what());
    return ACPF_EINVAL;
  }
  return ACPF_OK;
}

}  // extern "C"
