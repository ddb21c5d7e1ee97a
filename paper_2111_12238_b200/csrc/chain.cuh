// chain.cuh -- chain executor for the solve-family pairs (combos 1, 4, 8).
//
// A chain is a maximal run of consecutive rows (in processing order) where
// every row depends on the row right before it and on no other row closer
// than G positions.  In the reference summation order (ascending columns for
// the forward solve, descending for the backward L^T solve) the predecessor
// p-1 is always the LAST term, so
//     x_p = ((rhs - sum_{other deps} v x) - v_{p,p-1} x_{p-1}) / d_p
// splits into a partial sum that needs no value from the chain itself and a
// one-term carry.  A warp owns a chain: G lane groups compute the partial
// sums of G consecutive rows at once (all their loads in flight together),
// then the carry runs through the G rows with warp shuffles -- bit for bit
// the reference's arithmetic.  Chains are claimed in chain-DAG level order,
// a topological order, so every external dependency belongs to a chain that
// a running warp already owns.  On the 27-point grid a chain is one grid
// line: the x-direction part of the critical path never leaves the warp.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "internal.hpp"

namespace sfg {

struct ChainLayout {
  int32_t n = 0, G = 1, CS = 1, dir = +1;
  int32_t nchain = 0, nbatch = 0, nlevels = 0;
  DBuf<int32_t> cstart;    // chain -> first position (nchain + 1)
  DBuf<int32_t> corder;    // chains in claim order: (chain level, chain id)
  DBuf<int32_t> batch_ptr; // warp batch -> first index in corder (nbatch + 1)
  DBuf<int32_t> chain_of;  // position -> chain
  DBuf<int32_t> rank;      // chain -> index in corder
  DBuf<int32_t> clevel;    // chain -> chain-DAG level (tile skew)
  int64_t rows_chained = 0; // rows whose carry comes from the warp (stats)
};

// ptr/idx: CSR whose rows hold the dependencies in reference summation order
// followed by the diagonal; position p is row p (dir = +1) or row n-1-p
// (dir = -1).  G rows per tile, CS chains per warp.
void build_chains(const int32_t* ptr, const int32_t* idx, int32_t n, int dir, int32_t G,
                  int32_t CS, int32_t max_len, ChainLayout& out, cudaStream_t s);

// Combo 4: every SpMV row r becomes the "tail" of the forward chain that
// comes last in claim order among the chains it reads, so it runs as soon as
// that chain finishes (the paper's interleaved packing).
void build_tails(const ChainLayout& fwd, const int32_t* ar_ptr, const int32_t* ar_idx,
                 int32_t n, DBuf<int32_t>& tail_ptr, DBuf<int32_t>& tail_rows,
                 cudaStream_t s);

struct ChainArgs {
  int combo = 0;
  int32_t n = 0, S = 1;
  int32_t phase = 3; // bit 0: kernel-1 work, bit 1: kernel-2 work
  int32_t seg_begin = 0, seg_end = 0; // work items: [0, f_nbatch) fwd, then bwd
  unsigned long long* counter = nullptr;
  unsigned long long* err = nullptr;
  // forward solve (L rows, ascending)
  const int32_t *lr_ptr = nullptr, *lr_idx = nullptr;
  const double* lr_val = nullptr;
  const int32_t *f_cstart = nullptr, *f_corder = nullptr, *f_bptr = nullptr;
  const int32_t* f_level = nullptr;
  int32_t f_nbatch = 0;
  // backward solve (L' rows, descending)
  const int32_t *lt_ptr = nullptr, *lt_idx = nullptr;
  const double* lt_val = nullptr;
  const int32_t *b_cstart = nullptr, *b_corder = nullptr, *b_bptr = nullptr;
  const int32_t* b_level = nullptr;
  int32_t b_nbatch = 0;
  // combo 4 SpMV tails
  const int32_t *tail_ptr = nullptr, *tail_rows = nullptr;
  const int32_t *ar_ptr = nullptr, *ar_idx = nullptr;
  const double* ar_val = nullptr;
  // vectors
  const double* vin = nullptr;
  double* vmid = nullptr;
  double* vout = nullptr;
  int blocks_per_sm = 0;
  int tile_rows = 0; // tile height override (0 = chain_G's default)
  // tile skew per chain level, in rows: a chain at level l starts its tiles
  // (l * skew_mul) mod G rows early (1: a consumer tile needs the whole
  // same-index tile of its previous-level producers)
  int skew_mul = 1;
  // fused combo 8 (k_chain_sm): the backward outputs (vout, bwd_reset_words
  // 8-byte words) are reset in-kernel by the last bwd_reset_items forward
  // items; reset_done counts the finished slices (null: k_prep resets vout)
  double* bwd_reset = nullptr;
  int64_t bwd_reset_words = 0;
  int32_t bwd_reset_items = 0;
  unsigned long long* reset_done = nullptr;
  unsigned bwd_gate = 500; // ns a backward chain's first lane sleeps per check (0 = off)
  // optional timeline trace: per (work item, tile) {claim, partial done,
  // carry done} in %globaltimer ns (diagnostics only; null in production)
  unsigned long long* trace = nullptr;
  int32_t trace_tiles = 0;
};

// Tile geometry for S interleaved systems: G rows in flight per chain (one
// chain per warp).
// Tile height: 4 rows for S <= 8 systems, 32/S above.  Measured on C5
// (config 5's 27-point 128^3 fwd->bwd, ms per launch for S = 1 / 2 / 4 / 8):
// G = 2: 3.11 / 2.41 / 2.31 / 2.38; G = 4: 2.71 / 2.16 / 2.07 / 1.94;
// G = 8: 3.56 / 3.15 / 2.89 / -; G = 16: - / 5.40 / - / -.  Longer tiles
// lengthen the lag per chain level (paid at every one of the 382 levels),
// shorter ones the per-tile overhead; idle lanes at S < 8 cost little.
inline int32_t chain_G(int32_t S, int32_t override_rows = 0) {
  const int32_t g = S <= 8 ? 4 : 32 / S;
  return override_rows > 0 && override_rows * S <= 32 ? override_rows : g;
}
inline int32_t chain_CS(int32_t) { return 1; }

void launch_chain(const ChainArgs& a, cudaStream_t s);

} // namespace sfg
