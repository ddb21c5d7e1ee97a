// fact.cuh -- warp-per-task factorization executors (combos 5, 6, 7) driven
// by update lists the inspector precomputes (the symbolic phase).
//
// The reference finds, at run time, which finalized entries update a column
// (ic0_column, kernels.hpp:214-242: a marker array over column k and a scan
// of column j from L(k,j) on) or a row (ilu0_row, kernels.hpp:246-272).  That
// pattern depends only on the sparsity, so the inspector resolves it once
// into per-entry update lists, in the reference's order:
//   IC0:  position p of column k  ->  [(src, lkj)]  meaning  acc -= fac[lkj] * fac[src]
//         for each predecessor column j ascending (lkj = position of L(k,j))
//   ILU0: position p of row i     ->  [(step, src)] meaning  acc -= l_step * fac[src]
//         for each pivot step (lower entry k of row i, ascending)
// The executor then gives each task a warp and each factor entry a lane:
// all factor words a task needs are polled in one batch (one L2 round trip
// when they are ready), each lane applies its own few updates in order, the
// pivot quantities are exchanged by warp shuffles, and the fused solve row
// of kernel 2 is accumulated by lane 0 in the reference's order.
#pragma once

#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#include "executor.cuh"
#include "internal.hpp"

namespace sfg {

struct UpdateLists {
  DBuf<int32_t> ptr; // nnz(factor) + 1
  DBuf<int32_t> a;   // IC0: src position; ILU0: pivot step
  DBuf<int32_t> b;   // IC0: L(k,j) position; ILU0: src position (U(k,j))
  int64_t count = 0;
  int32_t max_task = 0;    // longest column / row (lanes needed)
  int32_t max_updates = 0; // most updates of one entry
  // packed executors (several same-level tasks per warp): SEG lanes per
  // task, packs of 32/SEG consecutive tickets inside one wavefront
  int32_t seg = 32;
  int32_t npack = 0;
  DBuf<int32_t> pack_ptr;
  // IC0 task records in claim order (8 ints per ticket), built at the first
  // fused launch of a combo-5 plan (k_ic0_pipe)
  mutable DBuf<int32_t> trec;
};

// combos 5, 7: L in CSC (lc_*) with its row view (rv_*)
void build_ic0_updates(const int32_t* lc_ptr, const int32_t* lc_idx, const int32_t* rv_ptr,
                       const int32_t* rv_col, const int32_t* rv_pos, int32_t n, int64_t nnz,
                       UpdateLists& out, cudaStream_t s);
// combos 3, 6: A in CSR (ar_*) with diagonal positions
void build_ilu0_updates(const int32_t* ar_ptr, const int32_t* ar_idx, const int32_t* diag,
                        int32_t n, int64_t nnz, UpdateLists& out, cudaStream_t s);

// Whether the warp executors cover every task of the plan (one lane per
// column / row entry; ILU0 keeps each entry's updates in registers).
// warps in one block of the factorization executors (occupancy sizing)
int fact_warps_per_block();
// Packs of 32/seg consecutive tickets that never cross a wavefront boundary
// (wave_ptr over the ticket order); sets up.seg / npack / pack_ptr.
void build_packs(const std::vector<int64_t>& wave_ptr, int32_t seg, UpdateLists& up);
bool ic0_warp_fits(const UpdateLists& up);
bool ilu0_warp_fits(const UpdateLists& up);

// Launches for one ticket range (ExecArgs as for the thread-per-task
// kernels); up = the update lists.
void launch_ic0_warp(int combo, const ExecArgs& a, const UpdateLists& up, cudaStream_t s);
void launch_ilu0_warp(int combo, const ExecArgs& a, const UpdateLists& up, cudaStream_t s);

} // namespace sfg
