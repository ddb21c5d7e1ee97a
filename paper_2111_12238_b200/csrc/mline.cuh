// mline.cuh -- multi-chain warp executor for the solve pairs (combos 1, 4, 8).
//
// A warp owns a GROUP of B = 32/S consecutive chains (chain = maximal run of
// positions whose last dependency is the previous position, see chain.cuh)
// and advances all of them in lockstep, one row per chain per STEP: at step i
// chain b computes its offset i - skew_b.  Lane (b, s) computes system s of
// chain b's row, so every lane is busy every step.  The inspector picks the
// skews so that every dependency on an earlier chain of the same group was
// produced at an earlier step; those values are read from a per-warp
// shared-memory ring (a few cycles) instead of being polled through L2 (a
// global hop, ~0.5 us).  Dependencies outside the group are gathered into
// shared memory by cp.async two steps ahead and re-polled only if they were
// still unpublished.  On the 27-point grid a group is B neighbouring grid
// lines, so the y-direction dependencies stay inside the warp and the group
// DAG has ~2.4x fewer levels than the line DAG.
//
// Arithmetic is the reference's: each row accumulates its dependencies in
// storage order (external or ring, whichever holds the value), then the
// carry term (always last), then divides -- bit for bit trsv_csr_row.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "chain.cuh"
#include "internal.hpp"

namespace sfg {

constexpr int32_t kRing = 8; // ring depth in steps (power of two)

struct MLineLayout {
  int32_t n = 0, S = 1, B = 32, dir = +1, CHN = 0;
  int32_t nchain = 0, ngroup = 0, nlevels = 0;
  int32_t max_steps = 0;
  int32_t est_steps = -1; // estimated makespan in steps (claim order by earliest start)
  DBuf<int32_t> cstart; // chain -> first position (nchain + 1)
  DBuf<int32_t> cskew;  // chain -> step of its offset 0 within the group
  DBuf<int32_t> gsteps; // group -> steps to run
  DBuf<int32_t> gorder; // groups in claim order (group-DAG level, id)
  DBuf<int32_t> glevel; // group -> group-DAG level (1-based)
  DBuf<int32_t> code;   // per CSR entry: >= 0 external row index, < 0 ring
                        // code -1 - (delta * 32 + b') (delta < kRing)
  DBuf<int32_t> chain_of; // position -> chain
  // Single-system step stream (S == 1, rows with <= kStreamChn dependencies):
  // group g's records start at sofs[g]; record sofs[g] + step * 32 + lane is
  // the row that lane computes at that step (srow, -1 = idle), its dependency
  // codes scode[rec][sch] (padding: external row n, the zero row) and
  // values sval[rec][sch + 4] (dependencies, carry coefficient, diagonal,
  // its reciprocal RN(1/d), padding), so a warp fetches a whole step with a
  // few coalesced copies.
  bool stream = false;
  int32_t sch = 4; // record width (2 or kStreamChn dependencies)
  int64_t nrec = 0;
  DBuf<int64_t> sofs;
  DBuf<int32_t> srow, scode;
  DBuf<double> sval;
};

constexpr int32_t kStreamChn = 4;

// (Re)builds the step stream from the current values (S == 1 only; sets
// L.stream = false when a row has more than kStreamChn dependencies).
void build_mline_stream(const int32_t* ptr, const double* val, int32_t n, int dir,
                        MLineLayout& L, cudaStream_t s);

// ptr/idx: CSR whose rows hold the dependencies in reference summation order
// followed by the diagonal; position p is row p (dir = +1) or row n-1-p
// (dir = -1).  B chains per group.
void build_mline(const int32_t* ptr, const int32_t* idx, int32_t n, int dir, int32_t S,
                 int32_t max_len, MLineLayout& out, cudaStream_t s);

// Widest dependency count (diagonal and carry excluded) over all rows.
int32_t mline_width(const int32_t* ptr, const int32_t* idx, int32_t n, int dir,
                    const MLineLayout& L, cudaStream_t s);

struct MLineArgs {
  int combo = 0;
  int32_t n = 0, S = 1;
  int32_t phase = 3;
  int32_t seg_begin = 0, seg_end = 0; // work items: [0, f_ngroup) fwd, then bwd
  unsigned long long* counter = nullptr;
  unsigned long long* err = nullptr;
  const int32_t *lr_ptr = nullptr, *lr_idx = nullptr;
  const double* lr_val = nullptr;
  const int32_t *f_cstart = nullptr, *f_cskew = nullptr, *f_gsteps = nullptr,
                *f_gorder = nullptr, *f_code = nullptr;
  int32_t f_nchain = 0, f_ngroup = 0;
  const int32_t *lt_ptr = nullptr, *lt_idx = nullptr;
  const double* lt_val = nullptr;
  const int32_t *b_cstart = nullptr, *b_cskew = nullptr, *b_gsteps = nullptr,
                *b_gorder = nullptr, *b_code = nullptr;
  int32_t b_nchain = 0, b_ngroup = 0;
  // combo 4: CSR(A) for the SpMV row blocks (b_ngroup = number of blocks)
  const int32_t *ar_ptr = nullptr, *ar_idx = nullptr;
  const double* ar_val = nullptr;
  const double* vin = nullptr;
  double* vmid = nullptr;
  double* vout = nullptr;
  int blocks_per_sm = 0;
  unsigned sleep_ns = 0; // back-off between re-polls of unpublished words
  int lookahead = 4;     // pipeline distance of the x gathers (2 or 4 steps)
  int32_t chn = 12; // staging width the kernel is instantiated for
  // step streams (k_mline1, S == 1): forward / second-segment layouts
  const int64_t *f_sofs = nullptr, *b_sofs = nullptr;
  const int32_t *f_srow = nullptr, *f_scode = nullptr, *b_srow = nullptr, *b_scode = nullptr;
  const double *f_sval = nullptr, *b_sval = nullptr;
  bool use_stream = false;
  int32_t stream_ch = 4;
  // diagnostics (SFG_TRACE): per work item {claim ns, first step ns, end ns,
  // stall cycles in cp.async waits << 32 | cycles in re-polls}
  unsigned long long* trace = nullptr;
};

// Largest staging width instantiated; wider rows read the excess directly.
constexpr int32_t kMLineMaxChn = 12;

void launch_mline(const MLineArgs& a, cudaStream_t s);

} // namespace sfg
