// Symbolic analysis result for the batched Newton engine (see nr_symbolic.cpp).
#pragma once
#include <cstdint>
#include <vector>

namespace acpf {

// Slot type bits (slot_type):
//   bit0  column unknown kind   0 = theta_j, 1 = V_j
//   bit1  row equation kind     0 = P_i,     1 = Q_i
//   bit2  diagonal bus block    i == j
//   8     fill (value starts at 0)
struct NrSymbolic {
  int n_bus = 0, n_theta = 0, n_q = 0, n_j = 0;
  int64_t nnz_y = 0, nnz_j = 0, nnz_lu = 0, n_pairs = 0;
  int etree_height = 0;
  std::vector<int32_t> perm;  // perm[p] = packed unknown at elimination position p
  std::vector<int32_t> ipos;  // inverse of perm
  std::vector<int32_t> row_bus, row_kind;
  std::vector<int64_t> rowptr, diag;
  std::vector<int32_t> col;
  std::vector<int32_t> slot_ynz, slot_jbus;
  std::vector<uint8_t> slot_type;
  std::vector<int64_t> pair_ptr;
  std::vector<int32_t> pair_l, pair_u;
};

void build_nr_symbolic(NrSymbolic& s, int n_bus, const int32_t* y_rowptr, const int32_t* y_col,
                       int n_theta, const int32_t* theta_block, int n_q, const int32_t* q_block,
                       const int32_t* perm_in);

}  // namespace acpf
