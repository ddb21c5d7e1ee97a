// executor.cuh -- argument block and launch entry points of the fused
// executor kernels (executor.cu).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace sfg {

// Everything one execution of a kernel pair touches.  Unused members are
// null for a given combo.  Numeric arrays of multi-system plans are
// interleaved (value[p * nsys + s], x[i * nsys + s]).
struct ExecArgs {
  int32_t n = 0;
  int32_t nsys = 1;
  int32_t phase = 3; // bit 0: kernel-1 work, bit 1: kernel-2 work
  const int32_t* order = nullptr;
  int64_t t_begin = 0, t_end = 0; // ticket range of this launch
  unsigned long long* counter = nullptr;
  // SFG_TRACE (factorization warps): per ticket {task, start, summed, fac
  // published, solve published} (globaltimer ns), 5 words
  unsigned long long* ftrace = nullptr;
  unsigned long long* err = nullptr;
  // L in CSR, diagonal last (trsv_csr_row, kernels.hpp:171-181)
  const int32_t* lr_ptr = nullptr;
  const int32_t* lr_idx = nullptr;
  const double* lr_val = nullptr;
  // L' rows = L columns reversed, diagonal last (combo 8 backward solve)
  const int32_t* lt_ptr = nullptr;
  const int32_t* lt_idx = nullptr;
  const double* lt_val = nullptr;
  // A in CSR (combo 4: row view of the CSC SpMV operand; combo 6: factor input)
  const int32_t* ar_ptr = nullptr;
  const int32_t* ar_idx = nullptr;
  const double* ar_val = nullptr;
  const int32_t* diag = nullptr;
  // L in CSC, diagonal first, plus its LowerRowView (kernels.hpp:86-115)
  const int32_t* lc_ptr = nullptr;
  const int32_t* lc_idx = nullptr;
  const double* lc_val = nullptr;
  const int32_t* rv_ptr = nullptr;
  const int32_t* rv_col = nullptr;
  const int32_t* rv_pos = nullptr;
  const double* dvec = nullptr;
  // vectors and outputs
  const double* vin = nullptr;
  double* vmid = nullptr;
  double* vout = nullptr;
  double* fac = nullptr;
  double* work = nullptr; // per-position scratch (long columns, DSCAL stage)
  unsigned sleep_cap = 160; // poll backoff cap in ns (0 = pure spin)
  int blocks_per_sm = 0;    // 0 = occupancy limit
};

struct FillRegion {
  void* ptr = nullptr;
  int64_t words = 0; // 8-byte words set to SENT
};

// Resets the ticket counter and error word and fills up to 3 regions with
// SENT, in one launch.
void launch_prep(const FillRegion* regions, int nregions,
                 unsigned long long* counter, unsigned long long* err,
                 cudaStream_t s);

// combo in {1, 4, 8}; nsys in {1, 2, 4, 8, 16, 32}.
void launch_trsv_pair(int combo, const ExecArgs& a, cudaStream_t s);
// combo in {5, 7}
void launch_ic0(int combo, const ExecArgs& a, cudaStream_t s);
// combo in {3, 6}
void launch_ilu0(int combo, const ExecArgs& a, cudaStream_t s);
// combo 3 kernel 1 alone (unfused): work[p] = (d_i * a_p) * d_j over CSR rows
void launch_dscal_csr(const ExecArgs& a, cudaStream_t s);
// combo 7 kernel 1 alone (unfused): work[p] = (d_i * a_p) * d_j
void launch_dscal(const ExecArgs& a, cudaStream_t s);
// execute_joint_wavefront (wavefront.cu): the joint level sets verts[lptr[l]
// .. lptr[l+1]) (vertex v < n: kernel-1 iteration v, else kernel-2 iteration
// v - n) level by level with a grid barrier between levels.  m_*: A in CSC
// for combo 4's scatter.  nlev < 0: run_sequential_reference on one thread.
void launch_wavefront(const ExecArgs& a, int combo, const int32_t* verts, const int64_t* lptr,
                      int32_t nlev, const int32_t* m_ptr, const int32_t* m_idx,
                      const double* m_val, cudaStream_t s);
// Number of violations of a flattened schedule (tags/iters on the host)
// against the joint DAG (successor CSR on the device, 2n vertices): an
// iteration missing or repeated, or an edge u -> v with v scheduled first.
int64_t check_schedule_order(const int32_t* jptr, const int32_t* jsucc, int32_t n,
                             const uint8_t* tags_h, const int32_t* iters_h, int64_t ne,
                             cudaStream_t s);

} // namespace sfg
