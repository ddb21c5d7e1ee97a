// bsf.cuh -- blocked sync-free (BSF) triangular-solve executor for the
// solve-family pairs (combos 1, 4, 8).
//
// The rows of a solve are cut into blocks of B consecutive rows in
// processing order (ascending for a forward solve, descending for the
// backward L^T solve).  One CTA owns a block at a time: inside the block the
// rows are ordered by their block-local wavefront, dependencies on rows of
// the same block are exchanged through shared memory (tens of cycles) and
// only dependencies on earlier blocks go through global memory (a polled
// word, ~0.5 us hop measured by scripts/micro_hop.cu).  Blocks are claimed
// in order from one ticket counter, so every awaited row is already owned by
// a running CTA.  This is the GPU form of the paper's fused partitioning:
// a block is a w-partition that runs without barriers, and the ticket order
// is the s-partition order -- without any global barrier.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>
#include <vector>

#include "internal.hpp"

namespace sfg {

// One solve's rows re-laid out in (block, local wavefront) order.
struct BsfLayout {
  int32_t n = 0, S = 1, B = 0, nblk = 0;
  int dir = +1;           // +1: positions are rows; -1: position p is row n-1-p
  DBuf<int32_t> rowP;     // slot -> row
  DBuf<int32_t> nptr;     // slot -> first strictly-triangular entry (n+1)
  DBuf<int32_t> nidx;     // >= 0: global row j; < 0: -(local slot + 1) in this block
  DBuf<double> nval;      // entry values, interleaved [e * S + s]
  DBuf<double> dval;      // diagonal, [slot * S + s]
  // Batches: runs of <= 32/S slots of one block-local wavefront.  A warp
  // processes whole batches, so its lanes never wait on each other.
  DBuf<int32_t> bptr;      // batch -> first slot (nbatch + 1)
  DBuf<int32_t> blk_batch; // block -> first batch (nblk + 1)
  int32_t nbatch = 0;
  int64_t nent = 0;
  int32_t max_local_levels = 0;
};

// Builds the layout from a CSR whose rows list their dependencies in the
// reference summation order with the diagonal last (L rows for the forward
// solve; L' rows, i.e. L columns reversed, for the backward solve).
void build_bsf(const int32_t* ptr, const int32_t* idx, const double* val,
               int32_t n, int32_t S, int dir, int32_t B, BsfLayout& out,
               cudaStream_t s);

// Ticket kinds (top 2 bits of a ticket word).
enum : int32_t { TK_FWD = 0, TK_BWD = 1, TK_Y = 2 };
inline int32_t ticket(int32_t kind, int32_t idx) { return (kind << 28) | idx; }

struct BsfArgs {
  int combo = 0;
  int32_t n = 0, S = 1;
  int32_t phase = 3;
  const int32_t* tickets = nullptr;
  int64_t nt = 0;
  unsigned long long* counter = nullptr;
  unsigned long long* err = nullptr;
  // forward layout (combos 1, 4, 8) and backward layout (combo 8)
  int32_t Bf = 0, nblk_f = 0;
  const int32_t *f_rowP = nullptr, *f_ptr = nullptr, *f_idx = nullptr;
  const double *f_val = nullptr, *f_diag = nullptr;
  const int32_t *f_bptr = nullptr, *f_blkb = nullptr;
  int32_t Bb = 0;
  const int32_t *b_rowP = nullptr, *b_ptr = nullptr, *b_idx = nullptr;
  const double *b_val = nullptr, *b_diag = nullptr;
  const int32_t *b_bptr = nullptr, *b_blkb = nullptr;
  // SpMV rows of combo 4 (CSR view of the CSC operand)
  int32_t By = 0;
  const int32_t *ar_ptr = nullptr, *ar_idx = nullptr;
  const double* ar_val = nullptr;
  // vectors
  const double* vin = nullptr;
  double* vmid = nullptr;
  double* vout = nullptr;
  int blocks_per_sm = 0;
};

// Ticket list for one fused execution (and the per-kernel ranges used by
// the unfused comparator).  Combo 4 interleaves each SpMV block right after
// the last forward block it reads (the paper's interleaved packing).
std::vector<int32_t> bsf_tickets(int combo, const BsfLayout& fwd,
                                 const BsfLayout* bwd, int32_t y_blocks,
                                 const std::vector<int32_t>& y_after_fwd_block,
                                 int64_t* k1_count);

void launch_bsf(const BsfArgs& a, cudaStream_t s);

} // namespace sfg
