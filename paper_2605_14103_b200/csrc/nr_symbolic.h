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

// Level-synchronous 2x2-block Crout schedule (see nr_kernel.cu).
//
// Unknowns are grouped per non-slack bus into 2x2 blocks [theta_i, V_i]
// (PV buses carry a padded V_i with the identity equation dV_i = 0), so the
// Jacobian is a block matrix with the Ybus pattern. The symbolic analysis
// (NrSymbolic) is run on that bus graph; its rows/slots are block rows/slots.
//
// Arena per scenario group: a block region of 4*kGroup-double elements
// (L^/U^ blocks, y/x 2-vectors padded to 4) followed by a
// scalar region of kGroup-double elements (per-bus phasors, state, specs).
struct NrSchedule {
  int64_t off_lu = 0, off_yx = 0, n_block = 0;                        // block region
  int64_t off_u = 0, off_e = 0, off_spec = 0, off_th = 0, off_vm = 0, n_scalar = 0;
  int max_l = 0;     // longest L part (blocks) of any row
  int n_levels = 0;  // factor levels (etree height)
  int n_blevels = 0; // back-substitution levels
  // per-bus assembly lists: entries asm_ptr[i]..asm_ptr[i+1]
  std::vector<int32_t> asm_ptr;
  std::vector<double> asm_y;      // [entries][2] Ybus value (0 for a missing diagonal)
  std::vector<int32_t> asm_j;     // [entries] column bus
  std::vector<int32_t> asm_slot;  // [entries] LU block slot (-1: slack column)
  std::vector<int32_t> bus_row;   // [n_bus] block row of the bus (-1 slack)
  // factor: rows are level-sorted; level l = rows level_ptr[l]..level_ptr[l+1]
  std::vector<int32_t> level_ptr, level_maxl;
  // warp tasks: consecutive rows of one level whose streams are processed by
  // one pipeline; tasks of level l are level_task_ptr[l]..level_task_ptr[l+1],
  // task k covers rows task_row[k]..task_row[k+1]
  std::vector<int32_t> level_task_ptr, task_row;
  std::vector<uint32_t> slot_info;  // [nnz_lu] flags | cnt << 16
  // storage position of each slot in the LU block region: U-part slots
  // (diagonal and right of it) column by column, then the L-part slots row by
  // row, so the U blocks one Crout target gathers (U_mc, m ascending) sit
  // next to each other in HBM
  std::vector<int32_t> slot_store;  // [nnz_lu]
  std::vector<int32_t> row_slot;    // [n_rows+1] = LU rowptr
  std::vector<int32_t> row_sptr;    // [n_rows+1] factor-row stream ranges
  // back substitution: rows in back order brow[r] = p | cnt << 20, grouped by
  // back level blevel_ptr; stream ranges brow_sptr (indexed by back position)
  std::vector<uint32_t> brow;
  std::vector<int32_t> blevel_ptr, brow_sptr;
  std::vector<int32_t> blevel_task_ptr, btask_row;  // same for back rows (back order)
  // gather stream, word = block element index | lpos << 22
  std::vector<uint32_t> stream;
  int64_t n_stream = 0;
  // Dense tail (nr_kernel.cu, nr_tail_kernel): the last tail_T block rows of
  // the level-sorted order (a suffix of whole levels, 2 tail_T <= 128). Their
  // Crout rows run as ONE factor level (tail_level) that only applies the
  // updates from non-tail rows and stores the partial values raw; the
  // on-chip dense LU of the tail (DMMA) finishes the factorisation, the
  // forward and the back substitution of the tail rows.
  int tail_row0 = 0;   // first tail row (= n_rows without a tail)
  int tail_T = 0;
  int tail_level = -1; // factor level of the tail rows, -1 without a tail
  // [slots][2]: storage element of a tail-column slot of a tail row, its
  // dense block position i * tail_T + j (i, j relative to tail_row0)
  std::vector<int32_t> tail_slot;
  // the tail level's tasks: one row each, grouped into classes by the length
  // of the row buffer they need (non-tail L blocks), one launch per class so
  // the short rows are not held to the occupancy of the longest one
  std::vector<int32_t> tail_trow, tail_class_ptr, tail_class_maxl;
};

constexpr uint32_t kSlotDiag = 1u << 5;
constexpr uint32_t kSlotRowEnd = 1u << 6;
constexpr uint32_t kSlotL = 1u << 8;
constexpr uint32_t kSlotFill = 1u << 9;
constexpr uint32_t kSlotTail = 1u << 10;  // tail-column slot of a tail row: store the partial value raw
#ifndef ACPF_TAIL_ROWS
#define ACPF_TAIL_ROWS 44
#endif
// 2 x kTailMaxRows scalar rows: one DMMA strip of 8 rows per warp. 44 (11 warps,
// 80 registers) lets two CTAs share an SM and overlap their latency-bound panel
// chains; 64 (16 warps) filled the register file with one scenario. gb2224 x
// 65,536: 64 -> 287.1 ms per solve, 48 -> 277.3, 44 -> 275.5, 40 -> 275.5,
// 36 -> 279.7, 32 -> 279.0 (one run, profiles/r2/nr_tail_kernel_phases.txt)
constexpr int kTailMaxRows = ACPF_TAIL_ROWS;

// s: NrSymbolic built on the non-slack buses (n_theta = #non-slack, n_q = 0)
void build_nr_schedule(const NrSymbolic& s, const int32_t* y_rowptr, const int32_t* y_col,
                       const double* y_re, const double* y_im, NrSchedule& out,
                       int task_elems = 512, bool column_store = true, int tail_max = 0);

// LU of the flat-start Jacobian, shared by the first Newton step of every
// scenario (see nr_symbolic.cpp); false on a zero pivot or non-finite value.
bool nr_flat_start_factor(const NrSymbolic& s, const NrSchedule& o, int n_bus, const int32_t* y_rowptr,
                          const int32_t* y_col, const double* y_re, const double* y_im, const int32_t* qidx,
                          const double* theta0, const double* vmag0, std::vector<double>& vals,
                          std::vector<double>* s0 = nullptr);

// Level-sorted topological reordering of an elimination order (same fill).
std::vector<int32_t> level_sorted_perm(const NrSymbolic& s);

// perm_in: elimination order (perm[k] = unknown eliminated k-th), or null to
// choose one: ordering 1 minimum degree, 2 minimum fill (kNrOrderMinFill)
constexpr int kNrOrderMinDegree = 1, kNrOrderMinFill = 2;
void build_nr_symbolic(NrSymbolic& s, int n_bus, const int32_t* y_rowptr, const int32_t* y_col,
                       int n_theta, const int32_t* theta_block, int n_q, const int32_t* q_block,
                       const int32_t* perm_in, int ordering = kNrOrderMinFill);

}  // namespace acpf
