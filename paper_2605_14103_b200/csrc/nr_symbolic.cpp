// Host-side symbolic analysis for the batched Newton solve (once per network).
//
// The reference never assembles the Jacobian (transmission.py:218-236 is a
// matrix-free JVP under FD-preconditioned GMRES, sparse.py:219-338). This
// engine replaces that step solve with an exact sparse LU, so it needs, once
// per network:
//   1. the Jacobian pattern implied by the Ybus pattern and the bus partition
//      (blocks H,N,M,L of dense_jacobian, transmission.py:383-407);
//   2. a fill-reducing symmetric ordering (built-in minimum degree, or the
//      caller's permutation);
//   3. the static-pivot L+U pattern (no pivoting: the probe in SURVEY.md 0.2
//      shows identical Newton flags/iterations to the reference);
//   4. per-slot assembly descriptors (which Ybus entry and which derivative
//      block feeds each LU slot; fill slots start at zero);
//   5. the Crout schedule: for every LU slot (p,c), the ordered list of
//      (l_pm, u_mc) slot pairs whose products are subtracted from a_pc.
// Everything here is plain C++; the device consumes the flat arrays.

#include "nr_symbolic.h"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <set>
#include <stdexcept>
#include <string>
#include <utility>

namespace acpf {

namespace {

// Eliminate the graph in `order`, or, if order is empty, choose the pivot
// greedily: kind 1 minimum degree, kind 2 minimum fill (fewest missing edges
// among the neighbours, then degree), lowest index breaking ties. Returns for
// each elimination step the neighbour set (original node ids) at elimination
// time = U-part of that row.
//
// Minimum fill is the default for the Newton plans: on the GB network it
// needs ~15% fewer block updates than MMD (the factor's gather stream) and a
// shallower elimination tree.
void eliminate(int n, std::vector<std::vector<int>>& adj, std::vector<int>& order,
               std::vector<std::vector<int>>& upart, int kind) {
  const bool choose = order.empty();
  std::vector<char> gone(n, 0);
  using Key = std::pair<std::pair<int64_t, int>, int>;  // ((fill or degree, degree), node)
  std::set<Key> pq;
  std::vector<Key> key(n);
  std::vector<int> mark(n, -1);
  int stamp = 0;
  auto score = [&](int v) -> Key {
    const auto& nv = adj[v];
    const int d = (int)nv.size();
    if (kind != 2) return {{d, d}, v};
    ++stamp;
    for (int a : nv) mark[a] = stamp;
    int64_t e2 = 0;  // 2 x edges among the neighbours
    for (int a : nv)
      for (int b : adj[a])
        if (mark[b] == stamp) ++e2;
    return {{(int64_t)d * (d - 1) / 2 - e2 / 2, d}, v};
  };
  if (choose) {
    order.reserve(n);
    for (int v = 0; v < n; ++v) pq.insert(key[v] = score(v));
  }
  upart.assign(n, {});
  std::vector<int> merged, touched;
  std::vector<int> tmark(n, -1);
  for (int k = 0; k < n; ++k) {
    int v;
    if (choose) {
      v = pq.begin()->second;
      pq.erase(pq.begin());
      order.push_back(v);
    } else {
      v = order[k];
      if (v < 0 || v >= n || gone[v]) throw std::invalid_argument("perm is not a permutation");
    }
    gone[v] = 1;
    std::vector<int> nb;
    nb.reserve(adj[v].size());
    for (int a : adj[v])
      if (!gone[a]) nb.push_back(a);
    // nb sorted (adj lists are kept sorted)
    for (int a : nb) {
      auto& la = adj[a];
      merged.clear();
      merged.reserve(la.size() + nb.size());
      std::set_union(la.begin(), la.end(), nb.begin(), nb.end(), std::back_inserter(merged));
      // drop a itself and v, and eliminated nodes
      la.clear();
      for (int b : merged)
        if (b != a && !gone[b]) la.push_back(b);
    }
    if (choose) {
      // rescore the neighbours (degree and fill change) and, for minimum
      // fill, their neighbours (edges among their neighbours changed)
      touched.clear();
      for (int a : nb) {
        if (tmark[a] != k) tmark[a] = k, touched.push_back(a);
        if (kind == 2)
          for (int b : adj[a])
            if (tmark[b] != k) tmark[b] = k, touched.push_back(b);
      }
      for (int a : touched) {
        pq.erase(key[a]);
        pq.insert(key[a] = score(a));
      }
    }
    upart[k] = std::move(nb);
    adj[v].clear();
    adj[v].shrink_to_fit();
  }
}

}  // namespace

void build_nr_symbolic(NrSymbolic& s, int n_bus, const int32_t* y_rowptr, const int32_t* y_col,
                       int n_theta, const int32_t* theta_block, int n_q, const int32_t* q_block,
                       const int32_t* perm_in, int ordering) {
  s.n_bus = n_bus;
  s.n_theta = n_theta;
  s.n_q = n_q;
  const int nj = n_theta + n_q;
  s.n_j = nj;
  if (nj <= 0) throw std::invalid_argument("no unknowns");

  std::vector<int> tpos(n_bus, -1), qpos(n_bus, -1);
  for (int k = 0; k < n_theta; ++k) {
    int b = theta_block[k];
    if (b < 0 || b >= n_bus || tpos[b] >= 0) throw std::invalid_argument("bad theta_block");
    tpos[b] = k;
  }
  for (int k = 0; k < n_q; ++k) {
    int b = q_block[k];
    if (b < 0 || b >= n_bus || qpos[b] >= 0) throw std::invalid_argument("bad q_block");
    if (tpos[b] < 0) throw std::invalid_argument("q_block bus missing from theta_block");
    qpos[b] = n_theta + k;
  }
  // packed unknown -> (bus, kind)
  std::vector<int> var_bus(nj), var_kind(nj);
  for (int k = 0; k < n_theta; ++k) var_bus[k] = theta_block[k], var_kind[k] = 0;
  for (int k = 0; k < n_q; ++k) var_bus[n_theta + k] = q_block[k], var_kind[n_theta + k] = 1;

  // J pattern (structurally symmetric): for unknown r at bus i, every bus j
  // with Y_ij present, plus j = i always.
  std::vector<std::vector<int>> adj(nj);
  s.nnz_y = y_rowptr[n_bus];
  for (int r = 0; r < nj; ++r) {
    int i = var_bus[r];
    auto add_bus = [&](int j) {
      if (tpos[j] >= 0 && tpos[j] != r) adj[r].push_back(tpos[j]);
      if (qpos[j] >= 0 && qpos[j] != r) adj[r].push_back(qpos[j]);
    };
    add_bus(i);
    for (int e = y_rowptr[i]; e < y_rowptr[i + 1]; ++e) {
      int j = y_col[e];
      if (j < 0 || j >= n_bus) throw std::invalid_argument("Ybus column out of range");
      add_bus(j);
    }
    std::sort(adj[r].begin(), adj[r].end());
    adj[r].erase(std::unique(adj[r].begin(), adj[r].end()), adj[r].end());
  }
  int64_t nnzj = nj;
  for (int r = 0; r < nj; ++r) nnzj += (int64_t)adj[r].size();
  s.nnz_j = nnzj;

  std::vector<int> order;
  if (perm_in) order.assign(perm_in, perm_in + nj);
  std::vector<std::vector<int>> upart;
  eliminate(nj, adj, order, upart, ordering);
  s.perm.assign(order.begin(), order.end());
  s.ipos.assign(nj, -1);
  for (int k = 0; k < nj; ++k) s.ipos[order[k]] = k;

  // rows in elimination order: U-part(k) in new positions; L-part by transpose
  std::vector<std::vector<int>> U(nj), L(nj);
  for (int k = 0; k < nj; ++k) {
    for (int a : upart[k]) U[k].push_back(s.ipos[a]);
    std::sort(U[k].begin(), U[k].end());
    for (int c : U[k]) L[c].push_back(k);  // k ascending => L[c] sorted
  }
  s.etree_height = 0;
  {
    std::vector<int> h(nj, 0);
    for (int k = 0; k < nj; ++k) {
      if (!U[k].empty()) {
        int par = U[k][0];
        h[par] = std::max(h[par], h[k] + 1);
      }
      s.etree_height = std::max(s.etree_height, h[k] + 1);
    }
  }

  // LU CSR (row-major, columns ascending: L-part, diag, U-part)
  s.rowptr.assign(nj + 1, 0);
  for (int p = 0; p < nj; ++p) s.rowptr[p + 1] = s.rowptr[p] + L[p].size() + 1 + U[p].size();
  const int64_t nslots = s.rowptr[nj];
  s.nnz_lu = nslots;
  s.col.resize(nslots);
  s.diag.resize(nj);
  for (int p = 0; p < nj; ++p) {
    int64_t t = s.rowptr[p];
    for (int m : L[p]) s.col[t++] = m;
    s.diag[p] = t;
    s.col[t++] = p;
    for (int c : U[p]) s.col[t++] = c;
  }

  // assembly descriptors: slot (p,c) = J[perm[p]][perm[c]]
  s.row_bus.resize(nj);
  s.row_kind.resize(nj);
  s.slot_ynz.assign(nslots, -2);
  s.slot_jbus.assign(nslots, 0);
  s.slot_type.assign(nslots, 0);
  std::vector<int64_t> where(nj, -1);
  for (int p = 0; p < nj; ++p) {
    int r = s.perm[p];
    int i = var_bus[r];
    s.row_bus[p] = i;
    s.row_kind[p] = var_kind[r];
    for (int64_t t = s.rowptr[p]; t < s.rowptr[p + 1]; ++t) where[s.col[t]] = t;
    auto put = [&](int j, int e) {
      // unknowns at bus j: theta (kind 0), V (kind 1)
      for (int kind = 0; kind < 2; ++kind) {
        int var = kind == 0 ? tpos[j] : qpos[j];
        if (var < 0) continue;
        int64_t t = where[s.ipos[var]];
        if (t < 0) throw std::logic_error("Jacobian entry missing from LU pattern");
        s.slot_ynz[t] = e;
        s.slot_jbus[t] = j;
        s.slot_type[t] = (uint8_t)(kind | (var_kind[r] << 1) | ((i == j) << 2));
      }
    };
    put(i, -1);  // diagonal bus block, y = 0 unless Y_ii present (below)
    for (int e = y_rowptr[i]; e < y_rowptr[i + 1]; ++e) put(y_col[e], e);
    for (int64_t t = s.rowptr[p]; t < s.rowptr[p + 1]; ++t) where[s.col[t]] = -1;
  }
  for (int64_t t = 0; t < nslots; ++t)
    if (s.slot_ynz[t] == -2) s.slot_type[t] = 8;  // fill

  // Crout schedule
  s.pair_ptr.assign(nslots + 1, 0);
  s.pair_l.clear();
  s.pair_u.clear();
  std::vector<std::vector<std::pair<int32_t, int32_t>>> lists;
  for (int p = 0; p < nj; ++p) {
    const int64_t r0 = s.rowptr[p], r1 = s.rowptr[p + 1];
    lists.assign(r1 - r0, {});
    for (int64_t t = r0; t < r1; ++t) where[s.col[t]] = t;
    for (int64_t tl = r0; tl < s.diag[p]; ++tl) {
      int m = s.col[tl];
      for (int64_t tu = s.diag[m] + 1; tu < s.rowptr[m + 1]; ++tu) {
        int c = s.col[tu];
        int64_t tt = where[c];
        if (tt < 0) throw std::logic_error("symbolic fill incomplete");
        lists[tt - r0].push_back({(int32_t)tl, (int32_t)tu});
      }
    }
    for (int64_t t = r0; t < r1; ++t) {
      where[s.col[t]] = -1;
      for (auto& pr : lists[t - r0]) {
        s.pair_l.push_back(pr.first);
        s.pair_u.push_back(pr.second);
      }
      s.pair_ptr[t + 1] = (int64_t)s.pair_l.size();
    }
  }
  s.n_pairs = (int64_t)s.pair_l.size();
  if (nslots > INT32_MAX || s.n_pairs > INT32_MAX)
    throw std::length_error("factor too large for 32-bit slot indices");
}

}  // namespace acpf

namespace acpf {

namespace {
std::vector<int> factor_levels(const NrSymbolic& s) {
  std::vector<int> lev(s.n_j, 0);
  for (int p = 0; p < s.n_j; ++p) {
    int l = 0;
    for (int64_t t = s.rowptr[p]; t < s.diag[p]; ++t) l = std::max(l, lev[s.col[t]] + 1);
    lev[p] = l;
  }
  return lev;
}
}  // namespace

std::vector<int32_t> level_sorted_perm(const NrSymbolic& s) {
  // rows of equal level never reference each other, and sorting by level is
  // a topological order of the elimination tree, so the filled pattern (and
  // nnz) is unchanged while rows that can be prefetched together become
  // contiguous.
  const std::vector<int> lev = factor_levels(s);
  std::vector<int32_t> idx(s.n_j);
  for (int p = 0; p < s.n_j; ++p) idx[p] = p;
  std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return lev[a] < lev[b]; });
  std::vector<int32_t> perm(s.n_j);
  for (int k = 0; k < s.n_j; ++k) perm[k] = s.perm[idx[k]];
  return perm;
}

void build_nr_schedule(const NrSymbolic& s, const int32_t* y_rowptr, const int32_t* y_col,
                       const double* y_re, const double* y_im, NrSchedule& o, int task_elems,
                       bool column_store, int tail_max) {
  const int nr = s.n_j, nb = s.n_bus;
  if (s.n_q != 0) throw std::logic_error("block schedule expects a bus-level symbolic analysis");
  // ---- arena layout
  o.off_lu = 0;
  o.off_yx = s.nnz_lu;
  o.n_block = o.off_yx + nr;
  int64_t e = 0;
  o.off_u = e;     e += 2 * (int64_t)nb;
  o.off_e = -1;    // no E = e^{j theta} vector: the Jacobian uses u_j / V_j
  o.off_spec = e;  e += 2 * (int64_t)nr;   // p_spec, q_spec per block row (0 for PV's q)
  o.off_th = e;    e += nb;
  o.off_vm = e;    e += nb;
  o.n_scalar = e;
  if (o.n_block >= (1 << 22)) throw std::length_error("block arena exceeds 22-bit gather index");
  o.max_l = 0;
  for (int p = 0; p < nr; ++p) o.max_l = std::max<int>(o.max_l, (int)(s.diag[p] - s.rowptr[p]));
  if (o.max_l >= 1024) throw std::length_error("L row longer than 1023 blocks");

  // ---- storage positions of the LU slots
  o.slot_store.assign(s.nnz_lu, 0);
  if (column_store) {
    std::vector<int64_t> ccount(nr + 1, 0);
    for (int p = 0; p < nr; ++p)
      for (int64_t t = s.diag[p]; t < s.rowptr[p + 1]; ++t) ++ccount[s.col[t] + 1];
    for (int c = 0; c < nr; ++c) ccount[c + 1] += ccount[c];
    int64_t nl = ccount[nr];
    for (int p = 0; p < nr; ++p) {  // rows ascending: each column's rows come out sorted
      for (int64_t t = s.rowptr[p]; t < s.diag[p]; ++t) o.slot_store[t] = (int32_t)nl++;
      for (int64_t t = s.diag[p]; t < s.rowptr[p + 1]; ++t)
        o.slot_store[t] = (int32_t)ccount[s.col[t]]++;
    }
  } else {
    for (int64_t t = 0; t < s.nnz_lu; ++t) o.slot_store[t] = (int32_t)t;
  }
  const std::vector<int32_t>& st = o.slot_store;

  // ---- bus -> block row, and per-bus assembly lists
  o.bus_row.assign(nb, -1);
  for (int p = 0; p < nr; ++p) o.bus_row[s.row_bus[p]] = p;
  std::vector<int64_t> where(nr, -1);
  o.asm_ptr.assign(nb + 1, 0);
  o.asm_y.clear();
  o.asm_j.clear();
  o.asm_slot.clear();
  for (int i = 0; i < nb; ++i) {
    const int p = o.bus_row[i];
    if (p >= 0) {
      for (int64_t t = s.rowptr[p]; t < s.rowptr[p + 1]; ++t) where[s.col[t]] = t;
      bool have_diag = false;
      for (int k = y_rowptr[i]; k < y_rowptr[i + 1]; ++k) have_diag |= (y_col[k] == i);
      auto emit = [&](int j, double yr, double yi) {
        int32_t slot = -1;
        if (o.bus_row[j] >= 0) {
          const int64_t t = where[o.bus_row[j]];
          if (t < 0) throw std::logic_error("assembly slot missing");
          slot = st[t];
        }
        o.asm_y.push_back(yr);
        o.asm_y.push_back(yi);
        o.asm_j.push_back(j);
        o.asm_slot.push_back(slot);
      };
      if (!have_diag) emit(i, 0.0, 0.0);
      for (int k = y_rowptr[i]; k < y_rowptr[i + 1]; ++k) emit(y_col[k], y_re[k], y_im[k]);
      for (int64_t t = s.rowptr[p]; t < s.rowptr[p + 1]; ++t) where[s.col[t]] = -1;
    }
    o.asm_ptr[i + 1] = (int32_t)o.asm_j.size();
  }

  // ---- levels (rows must already be level-sorted)
  std::vector<int> lev(nr, 0), blev(nr, 0);
  for (int p = 0; p < nr; ++p) {
    int l = 0;
    for (int64_t t = s.rowptr[p]; t < s.diag[p]; ++t) l = std::max(l, lev[s.col[t]] + 1);
    lev[p] = l;
    if (p && lev[p] < lev[p - 1]) throw std::logic_error("rows not level-sorted");
  }
  for (int p = nr - 1; p >= 0; --p) {
    int l = 0;
    for (int64_t t = s.diag[p] + 1; t < s.rowptr[p + 1]; ++t) l = std::max(l, blev[s.col[t]] + 1);
    blev[p] = l;
  }
  o.n_levels = lev[nr - 1] + 1;
  // ---- dense tail: the longest suffix of whole levels with at most
  // min(tail_max, kTailMaxRows) rows; those rows become one level
  {
    std::vector<int> cnt(o.n_levels, 0);
    for (int p = 0; p < nr; ++p) ++cnt[lev[p]];
    const int cap = std::min(tail_max, kTailMaxRows);
    int T = 0, l = o.n_levels - 1;
    while (l >= 0 && T + cnt[l] <= cap) T += cnt[l--];
    o.tail_T = T;
    o.tail_row0 = nr - T;
    o.tail_level = T > 0 ? l + 1 : -1;
    for (int p = o.tail_row0; p < nr; ++p) lev[p] = l + 1;
    if (T > 0) o.n_levels = l + 2;
  }
  const int n0 = o.tail_row0;
  // back levels of the non-tail rows: the tail's x is known before they run
  for (int p = nr - 1; p >= 0; --p) {
    int l = 0;
    if (p < n0)
      for (int64_t t = s.diag[p] + 1; t < s.rowptr[p + 1]; ++t)
        if (s.col[t] < n0) l = std::max(l, blev[s.col[t]] + 1);
    blev[p] = l;
  }
  o.n_blevels = 0;
  for (int p = 0; p < n0; ++p) o.n_blevels = std::max(o.n_blevels, blev[p] + 1);
  o.level_ptr.assign(o.n_levels + 1, 0);
  o.level_maxl.assign(o.n_levels, 0);
  for (int p = 0; p < nr; ++p) {
    o.level_ptr[lev[p] + 1] = p + 1;
    int nl = 0;  // L blocks kept in the row buffer (tail rows: the non-tail columns only)
    for (int64_t t = s.rowptr[p]; t < s.diag[p]; ++t) nl += (p < n0 || s.col[t] < n0) ? 1 : 0;
    o.level_maxl[lev[p]] = std::max<int>(o.level_maxl[lev[p]], nl);
  }

  // ---- factor stream: per block row b_p, then per slot: assembled block
  // (unless fill), the Crout updates' U^ blocks (with the L position), and for
  // an L slot y of its column (unit-upper form A = L^ U^, nr_kernel.cu)
  o.stream.clear();
  auto gw = [&](int64_t gidx, int lpos) {
    o.stream.push_back((uint32_t)gidx | ((uint32_t)lpos << 22));
  };
  o.slot_info.assign(s.nnz_lu, 0);
  o.row_slot.assign(nr + 1, 0);
  o.row_sptr.assign(nr + 1, 0);
  o.tail_slot.clear();
  for (int p = 0; p < nr; ++p) {
    const int64_t r0 = s.rowptr[p], r1 = s.rowptr[p + 1];
    o.row_slot[p + 1] = (int32_t)r1;
    gw(o.off_yx + p, 0);
    for (int64_t t = r0; t < r1; ++t) {
      // a tail row's slot in a tail column keeps only the updates from
      // non-tail rows m (pairs are in ascending m) and is stored raw
      const bool tail = p >= n0 && s.col[t] >= n0;
      uint32_t info = 0;
      if (tail) {
        info |= kSlotTail;
        o.tail_slot.push_back(st[t]);
        o.tail_slot.push_back((p - n0) * o.tail_T + (s.col[t] - n0));
      } else {
        if (t == s.diag[p]) info |= kSlotDiag;
        if (t < s.diag[p]) info |= kSlotL;
      }
      if (t == r1 - 1) info |= kSlotRowEnd;
      const bool fill = s.slot_type[t] == 8;
      if (fill) info |= kSlotFill;
      int64_t q1 = s.pair_ptr[t + 1];
      if (tail)
        for (q1 = s.pair_ptr[t]; q1 < s.pair_ptr[t + 1] && s.col[s.pair_l[q1]] < n0; ++q1) {
        }
      const int64_t cnt = q1 - s.pair_ptr[t];
      if (cnt >= 65536) throw std::length_error("too many updates for one slot");
      info |= (uint32_t)cnt << 16;
      o.slot_info[t] = info;
      if (!fill) gw(o.off_lu + st[t], 0);
      for (int64_t q = s.pair_ptr[t]; q < q1; ++q)
        gw(o.off_lu + st[s.pair_u[q]], (int)(s.pair_l[q] - r0));
      if (info & kSlotL) gw(o.off_yx + s.col[t], 0);  // y_t (unit-upper form: no pivot inverse)
    }
    o.row_sptr[p + 1] = (int32_t)o.stream.size();
  }
  // ---- back stream: rows by back level; per row y_p, then (U^_pc, x_c)
  // (tail rows are solved by the dense tail kernel and have no back rows)
  std::vector<int32_t> border(n0);
  for (int p = 0; p < n0; ++p) border[p] = p;
  std::stable_sort(border.begin(), border.end(), [&](int a, int b) {
    return blev[a] != blev[b] ? blev[a] < blev[b] : a > b;
  });
  o.brow.resize(n0);
  o.brow_sptr.assign(n0 + 1, 0);
  o.blevel_ptr.assign(o.n_blevels + 1, 0);
  o.brow_sptr[0] = (int32_t)o.stream.size();
  for (int r = 0; r < n0; ++r) {
    const int p = border[r];
    const int64_t cnt = s.rowptr[p + 1] - s.diag[p] - 1;
    if (p >= (1 << 20) || cnt >= 2048) throw std::length_error("back row too large");
    o.brow[r] = (uint32_t)p | ((uint32_t)cnt << 20);
    o.blevel_ptr[blev[p] + 1] = r + 1;
    gw(o.off_yx + p, 0);
    for (int64_t t = s.diag[p] + 1; t < s.rowptr[p + 1]; ++t) {
      gw(o.off_lu + st[t], 0);
      gw(o.off_yx + s.col[t], 0);
    }
    o.brow_sptr[r + 1] = (int32_t)o.stream.size();
  }
  o.n_stream = (int64_t)o.stream.size();
  if (o.n_stream >= INT32_MAX) throw std::length_error("stream too long");

  // ---- warp tasks: greedy runs of consecutive rows of one level with about
  // task_elems stream elements (a long row is a task on its own)
  auto make_tasks = [&](const std::vector<int32_t>& lptr, const std::vector<int32_t>& sptr,
                        std::vector<int32_t>& tptr, std::vector<int32_t>& trow) {
    const int nl = (int)lptr.size() - 1;
    tptr.assign(nl + 1, 0);
    trow.clear();
    for (int l = 0; l < nl; ++l) {
      int r = lptr[l];
      while (r < lptr[l + 1]) {
        trow.push_back(r);
        int64_t acc = 0;
        do {
          acc += sptr[r + 1] - sptr[r];
          ++r;
        } while (r < lptr[l + 1] && acc + (sptr[r + 1] - sptr[r]) <= task_elems);
      }
      tptr[l + 1] = (int32_t)trow.size();
    }
    trow.push_back(lptr[nl]);
  };
  make_tasks(o.level_ptr, o.row_sptr, o.level_task_ptr, o.task_row);
  o.tail_trow.clear();
  o.tail_class_ptr.assign(1, 0);
  o.tail_class_maxl.clear();
  if (o.tail_T > 0) {
    std::vector<int> nl(nr, 0);
    for (int p = n0; p < nr; ++p)
      for (int64_t t = s.rowptr[p]; t < s.diag[p]; ++t) nl[p] += s.col[t] < n0 ? 1 : 0;
    // row-buffer class bounds (L blocks); ACPF_NR_TAIL_CLASSES="b1,b2,..." overrides
    std::vector<int> bounds = {16, 32, 48, 64};
    if (const char* env = std::getenv("ACPF_NR_TAIL_CLASSES")) {
      bounds.clear();
      for (const char* c = env; *c;) {
        char* end = nullptr;
        const long v = std::strtol(c, &end, 10);
        if (end == c) break;
        if (v > 0) bounds.push_back((int)v);
        c = (*end == ',') ? end + 1 : end;
      }
      std::sort(bounds.begin(), bounds.end());
    }
    bounds.push_back(1 << 30);
    int lo = -1;
    for (int hi : bounds) {
      int mx = 0;
      for (int p = n0; p < nr; ++p)
        if (nl[p] > lo && nl[p] <= hi) {
          o.tail_trow.push_back(p);
          mx = std::max(mx, nl[p]);
        }
      if ((int)o.tail_trow.size() > o.tail_class_ptr.back()) {
        o.tail_class_ptr.push_back((int)o.tail_trow.size());
        o.tail_class_maxl.push_back(mx);
      }
      lo = hi;
    }
  }
  make_tasks(o.blevel_ptr, o.brow_sptr, o.blevel_task_ptr, o.btask_row);
}

// The Jacobian at the flat start (transmission.py:169-177) depends only on
// the network and the flat-start state, never on the specified injections, so
// the first Newton step of every scenario factors the same matrix. It is
// assembled here with the device formulas (nr_mismatch_kernel: dense_jacobian,
// transmission.py:383-407, PV padding rows/columns dV = 0) and factored once in
// the same unit-upper block form as nr_factor_kernel (Crout pair lists of s).
// vals[4t + 2i + j] = entry (i, j) of slot t: L^ for L slots, inv(D_p) at the
// diagonal slot, U^ = inv(D_p) A' for U slots. Returns false on an exact zero
// pivot (the caller then factors step 0 per scenario as in every other step).
bool nr_flat_start_factor(const NrSymbolic& s, const NrSchedule& o, int n_bus, const int32_t* y_rowptr,
                          const int32_t* y_col, const double* y_re, const double* y_im, const int32_t* qidx,
                          const double* theta0, const double* vmag0, std::vector<double>& vals,
                          std::vector<double>* s0) {
  const int nr = s.n_j;
  const int64_t nslots = s.rowptr[nr];
  std::vector<double> er(n_bus), ei(n_bus), ur(n_bus), ui(n_bus);
  for (int i = 0; i < n_bus; ++i) {
    er[i] = std::cos(theta0[i]);
    ei[i] = std::sin(theta0[i]);
    ur[i] = vmag0[i] * er[i];
    ui[i] = vmag0[i] * ei[i];
  }
  std::vector<double> a(4 * nslots, 0.0);
  std::vector<int64_t> where(nr, -1);
  if (s0) s0->assign(2 * (size_t)n_bus, 0.0);
  for (int i = 0; i < n_bus; ++i) {
    const int p = o.bus_row[i];
    if (p < 0) continue;
    double ir = 0.0, ii = 0.0;  // I_i = sum_j Y_ij u_j
    for (int e = y_rowptr[i]; e < y_rowptr[i + 1]; ++e) {
      const int j = y_col[e];
      ir += y_re[e] * ur[j] - y_im[e] * ui[j];
      ii += y_re[e] * ui[j] + y_im[e] * ur[j];
    }
    if (s0) {  // S_i = u_i conj(I_i) at the flat start (the step-0 mismatch of every scenario)
      (*s0)[2 * i] = ur[i] * ir + ui[i] * ii;
      (*s0)[2 * i + 1] = ui[i] * ir - ur[i] * ii;
    }
    for (int64_t t = s.rowptr[p]; t < s.rowptr[p + 1]; ++t) where[s.col[t]] = t;
    const bool pq = qidx[i] >= 0;
    auto stamp = [&](int j, double yr, double yi) {
      if (o.bus_row[j] < 0) return;  // slack column
      const int64_t t = where[o.bus_row[j]];
      if (t < 0) throw std::logic_error("flat-start assembly slot missing");
      // wv = u_i conj(y E_j)
      const double ye_r = yr * er[j] - yi * ei[j], ye_i = yr * ei[j] + yi * er[j];
      const double wvr = ur[i] * ye_r + ui[i] * ye_i, wvi = ui[i] * ye_r - ur[i] * ye_i;
      double dthr, dthi, dvr, dvi;
      if (j != i) {  // dS_i/dth_j = -j u_i conj(y u_j)
        const double yu_r = yr * ur[j] - yi * ui[j], yu_i = yr * ui[j] + yi * ur[j];
        const double wtr = ur[i] * yu_r + ui[i] * yu_i, wti = ui[i] * yu_r - ur[i] * yu_i;
        dthr = wti;
        dthi = -wtr;
        dvr = wvr;
        dvi = wvi;
      } else {  // dS_i/dth_i = j u_i conj(I_i - y u_i); dS_i/dV_i = wv + conj(I_i) E_i
        const double yu_r = yr * ur[i] - yi * ui[i], yu_i = yr * ui[i] + yi * ur[i];
        const double cr = ir - yu_r, ci = ii - yu_i;
        const double wtr = ur[i] * cr + ui[i] * ci, wti = ui[i] * cr - ur[i] * ci;
        dthr = -wti;
        dthi = wtr;
        dvr = wvr + (ir * er[i] + ii * ei[i]);
        dvi = wvi + (ir * ei[i] - ii * er[i]);
      }
      const bool pqj = qidx[j] >= 0;
      double* b = &a[4 * t];
      b[0] = dthr;                                           // H
      b[2] = pq ? dthi : 0.0;                                // M
      b[1] = pqj ? dvr : 0.0;                                // N
      b[3] = (pq && pqj) ? dvi : (j == i ? 1.0 : 0.0);       // L (PV padding: dV = 0)
    };
    bool have_diag = false;
    for (int e = y_rowptr[i]; e < y_rowptr[i + 1]; ++e) have_diag |= (y_col[e] == i);
    if (!have_diag) stamp(i, 0.0, 0.0);
    for (int e = y_rowptr[i]; e < y_rowptr[i + 1]; ++e) stamp(y_col[e], y_re[e], y_im[e]);
    for (int64_t t = s.rowptr[p]; t < s.rowptr[p + 1]; ++t) where[s.col[t]] = -1;
  }
  vals.assign(4 * nslots, 0.0);
  for (int p = 0; p < nr; ++p) {
    double inv[4] = {0, 0, 0, 0};
    for (int64_t t = s.rowptr[p]; t < s.rowptr[p + 1]; ++t) {
      double c[4] = {a[4 * t], a[4 * t + 1], a[4 * t + 2], a[4 * t + 3]};
      for (int64_t k = s.pair_ptr[t]; k < s.pair_ptr[t + 1]; ++k) {
        const double* l = &vals[4 * (int64_t)s.pair_l[k]];
        const double* u = &vals[4 * (int64_t)s.pair_u[k]];
        for (int i = 0; i < 2; ++i)
          for (int j = 0; j < 2; ++j) c[2 * i + j] -= l[2 * i] * u[j] + l[2 * i + 1] * u[2 + j];
      }
      double* v = &vals[4 * t];
      if (t < s.diag[p]) {
        for (int k = 0; k < 4; ++k) v[k] = c[k];
      } else if (t == s.diag[p]) {
        const double det = c[0] * c[3] - c[1] * c[2];
        if (det == 0.0 || !std::isfinite(det)) return false;
        const double rd = 1.0 / det;
        inv[0] = c[3] * rd;
        inv[1] = -c[1] * rd;
        inv[2] = -c[2] * rd;
        inv[3] = c[0] * rd;
        for (int k = 0; k < 4; ++k) v[k] = inv[k];
      } else {
        for (int i = 0; i < 2; ++i)
          for (int j = 0; j < 2; ++j) v[2 * i + j] = inv[2 * i] * c[j] + inv[2 * i + 1] * c[2 + j];
      }
    }
  }
  for (double x : vals)
    if (!std::isfinite(x)) return false;
  return true;
}

}  // namespace acpf
