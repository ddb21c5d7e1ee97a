// ell.cuh -- chain-ELL layout and the TMA-staged chain executor for batched
// solves (S >= 2 interleaved systems; combo 8 forward L then backward L').
//
// Layout (built by the inspector from the chain decomposition, chain.cuh):
// every position p of a solve gets a fixed-width record
//     eidx[p][CHN]               dependency rows (reference order, carry
//                                excluded), padded with the zero row n
//     eval[p][CHN + 2][S]        their values (padding 0.0), then the carry
//                                coefficient v_{p,p-1} (0 at a chain start),
//                                then the diagonal
// so a tile of G consecutive positions is one contiguous byte range.  A
// padded term adds 0.0 * (+0.0) = +0.0 and acc - (+0.0) == acc exactly, so
// the arithmetic stays the reference's bit for bit.  The x vectors carry an
// extra all-zero row n that the padding points at.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "chain.cuh"
#include "internal.hpp"

namespace sfg {

struct EllLayout {
  int32_t n = 0, S = 1, CHN = 0, dir = +1;
  DBuf<int32_t> eidx; // n * CHN
  DBuf<double> eval;  // n * (CHN + 2) * S
};

// Widest non-carry dependency count of any position (0 if n == 0).
int32_t ell_width(const int32_t* ptr, const int32_t* idx, int32_t n, int dir,
                  const ChainLayout& ch, cudaStream_t s);

// Builds the layout; CHN must be >= ell_width and a multiple of 4.
void build_ell(const int32_t* ptr, const int32_t* idx, const double* val, int32_t n, int32_t S,
               int dir, int32_t CHN, const ChainLayout& ch, EllLayout& out, cudaStream_t s);

struct EllArgs {
  int32_t n = 0, S = 1;
  int32_t seg_begin = 0, seg_end = 0;
  unsigned long long* counter = nullptr;
  unsigned long long* err = nullptr;
  // forward (fwd) and backward (bwd) chain schedules and layouts
  const int32_t *f_cstart = nullptr, *f_corder = nullptr, *f_bptr = nullptr, *f_level = nullptr;
  int32_t f_nbatch = 0;
  const int32_t* f_eidx = nullptr;
  const double* f_eval = nullptr;
  const int32_t *b_cstart = nullptr, *b_corder = nullptr, *b_bptr = nullptr, *b_level = nullptr;
  const int32_t* b_eidx = nullptr;
  const double* b_eval = nullptr;
  const double* vin = nullptr;
  double* vmid = nullptr; // n + 1 rows (row n all zero)
  double* vout = nullptr; // n + 1 rows (row n all zero)
  int warps_per_cta = 4;
  int blocks_per_sm = 0;
  int ws_slots = 3; // warp-specialised executor: slots per warp pair (2 or 3)
  int ws_pairs = 2; // warp pairs per CTA (more CTAs per SM fit when small)
  int ws_fence = 0; // diagnostics: fence after each tile's publishes
  // diagnostics: completion time (globaltimer ns) of tile u of work item i
  // at trace[i * trace_tiles + u]; null in production
  unsigned long long* trace = nullptr;
  int32_t trace_tiles = 0;
};

// Largest CHN the TMA executor is compiled for.
constexpr int32_t kEllMaxWidth = 16;

void launch_chain_ell(const EllArgs& a, int32_t CHN, cudaStream_t s);

// Warp-specialised variant (chainws.cu): a loader warp and a compute warp per
// chain share a ring of shared-memory slots.  Combo 8, S in {4, 8, 16, 32}.
void launch_chain_ws(const EllArgs& a, int32_t CHN, cudaStream_t s);

} // namespace sfg
