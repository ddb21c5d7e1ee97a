// plan.cu -- the C-ABI (include/sfgpu.h): plan = a KernelState resident in
// HBM plus its GPU-built schedule.  Mirrors make_state / build_g1 / build_g2
// / inter_dag / joint_dag / level_info / compute_reuse / execute_fused /
// execute_unfused / collect_outputs (kernels.hpp, dag.hpp, executor.hpp).
#include "../../include/sfgpu.h"
#include "chain.cuh"
#include "fact.cuh"
#include "mline.cuh"
#include "common.cuh"
#include "executor.cuh"
#include "internal.hpp"

#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <memory>
#include <random>
#include <cmath>
#include <string>
#include <vector>

using namespace sfg;

struct sfg_plan {
  int combo = 0;
  int32_t n = 0;
  int32_t nsys = 1;
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t own_stream = nullptr;
  int64_t launches = 0;
  int64_t nnzM = 0, nnzL = 0, nnzF = 0; // M, lower(M), factor outputs
  int64_t lower_count = 0;

  DBuf<int32_t> m_ptr, m_idx; // M pattern (CSC)
  DBuf<double> m_val;         // M values (combo 4: the wavefront executor's CSC scatter)
  DBuf<int32_t> lr_ptr, lr_idx;
  DBuf<double> lr_val;
  DBuf<int32_t> lt_ptr, lt_idx;
  DBuf<double> lt_val;
  DBuf<int32_t> ar_ptr, ar_idx, diag;
  DBuf<double> ar_val;
  DBuf<int32_t> lc_ptr, lc_idx, rv_ptr, rv_col, rv_pos;
  DBuf<double> lc_val, dvec;
  DBuf<double> vin, vmid, vout, fac, work, staging;
  // value maps (positions in M) kept for sfg_set_values
  DBuf<int32_t> map_lc, map_lr, map_lt, map_ar;
  DBuf<double> mstage;

  // schedule
  bool inspected = false;
  DBuf<int32_t> order;
  int64_t ntickets = 0;
  std::vector<int64_t> wave_ptr; // wavefront boundaries over tickets
  int32_t seg2_start_wave = -1;  // first wave of the second ticket segment
  DBuf<unsigned long long> counter, err;

  // joint-DAG level sets (build_wavefront_schedule) for the wavefront executor
  bool have_wf = false;
  DBuf<int32_t> wf_verts;
  DBuf<int64_t> wf_lptr;
  std::vector<int64_t> wf_ptr;

  // parity structures (lazy)
  std::unique_ptr<DevDag> dags[3];
  std::unique_ptr<DevDag> fdep;
  DBuf<int32_t> lev[3], hgt[3], slk[3];
  int32_t crit[3] = {0, 0, 0};
  bool have_levels[3] = {false, false, false};

  // chain executor (combos 1, 4, 8); the level-set kernel stays available
  // as SFG_EXECUTOR=levels for ablations
  bool use_chain = false;
  ChainLayout ch_f, ch_b;
  DBuf<int32_t> tail_ptr, tail_rows;
  std::vector<int32_t> row_maxcol; // (unused by the chain path; kept for stats)
  int32_t tile_rows = 0;           // chain tile height override (0 = chain_G default)
  DBuf<unsigned long long> trace;  // SFG_TRACE diagnostics
  // multi-chain warp executor (combos 1, 8; default)
  bool use_mline = false;
  MLineLayout ml_f, ml_b;
  // warp-per-task factorization executors (combos 5, 6, 7)
  bool use_warpfac = false;
  UpdateLists upd;
  int32_t trace_tiles = 0;

  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  // sfg_execute_batch: copy streams, double-buffered host-facing staging
  cudaStream_t copy_in = nullptr, copy_out = nullptr;
  DBuf<double> in_stage[2], out_stage[2];
  DBuf<unsigned long long> err_hist;
  cudaEvent_t bev[8] = {};
  bool timed = false;

  // last error
  int32_t ferr_kind = 0, ferr_index = -1;
  std::string msg;
};

namespace {

struct LaunchScope {
  int64_t* prev;
  explicit LaunchScope(sfg_plan* p) : prev(g_launch_counter) { g_launch_counter = &p->launches; }
  ~LaunchScope() { g_launch_counter = prev; }
};

struct DeviceScope {
  int prev = 0;
  explicit DeviceScope(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev)
      cudaSetDevice(dev);
  }
  ~DeviceScope() {
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != prev)
      cudaSetDevice(prev);
  }
};

sfg_status set_err(sfg_plan* p, sfg_status st, const std::string& m, int32_t kind = 0,
                   int32_t index = -1) {
  if (p) {
    p->msg = m;
    p->ferr_kind = kind;
    p->ferr_index = index;
  }
  return st;
}

template <typename F> sfg_status guarded(sfg_plan* p, F&& f) {
  try {
    return f();
  } catch (const InvalidMatrix& e) {
    return set_err(p, SFG_ERR_INVALID_MATRIX, e.what(), SFG_FERR_INVALID_MATRIX, e.index);
  } catch (const InvalidArgument& e) {
    return set_err(p, SFG_ERR_INVALID_ARGUMENT, e.what());
  } catch (const FactorizationFailure& e) {
    return set_err(p, SFG_ERR_FACTORIZATION, e.what(), e.kind, e.index);
  } catch (const CudaError& e) {
    return set_err(p, SFG_ERR_CUDA, e.what());
  } catch (const std::bad_alloc&) {
    return set_err(p, SFG_ERR_CUDA, "host allocation failed");
  } catch (const std::exception& e) {
    return set_err(p, SFG_ERR_LOGIC, e.what());
  }
}

inline unsigned grid_for(int64_t work, int block = 256) {
  int64_t g = (work + block - 1) / block;
  const int64_t cap = (int64_t)sm_count() * 32;
  if (g > cap)
    g = cap;
  return (unsigned)(g < 1 ? 1 : g);
}

template <typename T> void upload(DBuf<T>& d, const T* h, int64_t n, cudaStream_t s) {
  d.alloc(n > 0 ? n : 1);
  if (n > 0)
    SFG_CUDA(cudaMemcpyAsync(d.p, h, sizeof(T) * (size_t)n, cudaMemcpyHostToDevice, s));
}

__global__ void compose_kernel(const int32_t* __restrict__ a, const int32_t* __restrict__ b,
                               int64_t n, int32_t* __restrict__ out) {
  // out[q] = a[b[q]]
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x)
    out[q] = a[b[q]];
}

// LowerRowView from the CSR of L (diagonal last per row): drop each row's
// last entry; row i shifts left by i (kernels.hpp:92-115).
__global__ void rowview_kernel(const int32_t* __restrict__ csr_ptr,
                               const int32_t* __restrict__ csr_idx,
                               const int32_t* __restrict__ perm, int32_t n,
                               int32_t* __restrict__ rv_ptr, int32_t* __restrict__ rv_col,
                               int32_t* __restrict__ rv_pos) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= n;
       i += (int64_t)gridDim.x * blockDim.x) {
    rv_ptr[i] = csr_ptr[i] - (int32_t)i;
    if (i < n)
      for (int32_t q = csr_ptr[i]; q < csr_ptr[i + 1] - 1; ++q) {
        rv_col[q - i] = csr_idx[q];
        rv_pos[q - i] = perm[q];
      }
  }
}

__global__ void iota_i32_kernel(int32_t* a, int64_t n, int32_t base) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    a[i] = base + (int32_t)i;
}

// Edge-key generators for the parity DAGs (dag.hpp:150-192, 222-238,
// 279-317).  Every entry of a compressed structure yields one key (u<<32|v)
// or the all-ones "no edge" key.
enum EdgeMode {
  EM_ROWS_LOWER = 0, // CSR rows: (col, row) if col < row
  EM_COLS_BELOW = 1, // CSC columns: (col, row) if row > col
  EM_LT_REV = 2,     // L' rows (orig i): (n-1-j, n-1-i) if j > i
  EM_SUCC = 3,       // generic successor CSR with offsets
  EM_FDEP = 4        // F rows i: (col, off_v + i)
};

__global__ void edge_keys_kernel(const int32_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                                 int32_t nmajor, int mode, int32_t n, int32_t off_u,
                                 int32_t off_v, uint64_t* __restrict__ keys) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int32_t base = ptr[0];
  for (int64_t m = warp; m < nmajor; m += nwarps) {
    for (int32_t p = ptr[m] + lane; p < ptr[m + 1]; p += 32) {
      const int32_t x = idx[p];
      uint64_t key = ~0ull;
      int64_t u = -1, v = -1;
      switch (mode) {
      case EM_ROWS_LOWER:
        if (x < m) {
          u = x;
          v = m;
        }
        break;
      case EM_COLS_BELOW:
        if (x > m) {
          u = m;
          v = x;
        }
        break;
      case EM_LT_REV:
        if (x > m) {
          u = n - 1 - x;
          v = n - 1 - m;
        }
        break;
      case EM_SUCC:
        u = m + off_u;
        v = x + off_v;
        break;
      case EM_FDEP:
        u = x;
        v = off_v + m;
        break;
      }
      if (u >= 0)
        key = ((uint64_t)u << 32) | (uint64_t)v;
      keys[p - base] = key;
    }
  }
}

enum CostKind {
  CK_ROWNNZ = 0,   // max(1, ptr[i+1]-ptr[i])  (SpTRSV_CSR, SpMV/DSCAL_CSC)
  CK_IC0 = 1,      // dag.hpp:128-140
  CK_TRSV_CSC = 2, // 1 + row-view count
  CK_ILU0 = 3,     // dag.hpp:92-105
  CK_UNIT = 4,     // combo 6 G2: 1 + strictly-lower count
  CK_LT_REV = 5    // combo 8 G2: cost[n-1-i] = max(1, L' row length)
};

__global__ void cost_kernel(int kind, int32_t n, const int32_t* __restrict__ ptr,
                            const int32_t* __restrict__ idx, const int32_t* __restrict__ ptr2,
                            const int32_t* __restrict__ aux1, const int32_t* __restrict__ aux2,
                            int64_t* __restrict__ cost) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t c = 0;
    switch (kind) {
    case CK_ROWNNZ:
      c = max((int64_t)1, (int64_t)(ptr[i + 1] - ptr[i]));
      break;
    case CK_IC0: { // ptr = lc_ptr, ptr2 = rv_ptr, aux1 = rv_col, aux2 = rv_pos
      int64_t t = ptr[i + 1] - ptr[i];
      for (int32_t q = ptr2[i]; q < ptr2[i + 1]; ++q)
        t += ptr[aux1[q] + 1] - aux2[q];
      c = max((int64_t)1, t);
      break;
    }
    case CK_TRSV_CSC: // ptr2 = rv_ptr
      c = 1 + ptr2[i + 1] - ptr2[i];
      break;
    case CK_ILU0: { // ptr/idx = A_csr, aux1 = diag
      int64_t t = ptr[i + 1] - ptr[i];
      for (int32_t p = ptr[i]; p < ptr[i + 1]; ++p) {
        const int32_t k = idx[p];
        if (k >= i)
          break;
        if (aux1[k] >= 0)
          t += ptr[k + 1] - aux1[k] - 1;
      }
      c = max((int64_t)1, t);
      break;
    }
    case CK_UNIT: {
      int64_t t = 1;
      for (int32_t p = ptr[i]; p < ptr[i + 1]; ++p) {
        if (idx[p] >= i)
          break;
        ++t;
      }
      c = t;
      break;
    }
    case CK_LT_REV:
      cost[n - 1 - i] = max((int64_t)1, (int64_t)(ptr[i + 1] - ptr[i]));
      continue;
    }
    cost[i] = c;
  }
}

__global__ void fdep_fill_kernel(int combo, int32_t n, const int32_t* __restrict__ m_ptr,
                                 const int32_t* __restrict__ rv_ptr,
                                 const int32_t* __restrict__ rv_col,
                                 const int32_t* __restrict__ ar_ptr,
                                 const int32_t* __restrict__ ar_idx,
                                 const int32_t* __restrict__ rowptr, int32_t* __restrict__ colidx) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t w = rowptr[i];
    switch (combo) {
    case 1:
    case 2:
    case 6:
      colidx[w] = (int32_t)i;
      break;
    case 3: // dag.hpp:294-302: the DSCAL rows k <= i of A's row i
      for (int32_t p = ar_ptr[i]; p < ar_ptr[i + 1] && ar_idx[p] <= i; ++p)
        colidx[w++] = ar_idx[p];
      break;
    case 8:
      colidx[w] = n - 1 - (int32_t)i;
      break;
    case 4:
      if (m_ptr[i] < m_ptr[i + 1])
        colidx[w] = (int32_t)i;
      break;
    case 5:
    case 7:
      for (int32_t q = rv_ptr[i]; q < rv_ptr[i + 1]; ++q)
        colidx[w++] = rv_col[q];
      colidx[w] = (int32_t)i;
      break;
    }
  }
}

__global__ void fdep_count_kernel(int combo, int32_t n, const int32_t* __restrict__ m_ptr,
                                  const int32_t* __restrict__ rv_ptr,
                                  const int32_t* __restrict__ ar_ptr,
                                  const int32_t* __restrict__ ar_idx, int32_t* __restrict__ cnt) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i == n) {
      cnt[i] = 0;
      continue;
    }
    int32_t c = 1;
    if (combo == 4)
      c = m_ptr[i] < m_ptr[i + 1] ? 1 : 0;
    else if (combo == 5 || combo == 7)
      c = rv_ptr[i + 1] - rv_ptr[i] + 1;
    else if (combo == 3) {
      c = 0;
      for (int32_t p = ar_ptr[i]; p < ar_ptr[i + 1] && ar_idx[p] <= i; ++p)
        ++c;
    }
    cnt[i] = c;
  }
}

__global__ void collect_pair_kernel(const double* __restrict__ vmid, const double* __restrict__ vout,
                                    int32_t n, int32_t nsys, double* __restrict__ out) {
  const int64_t total = (int64_t)n * nsys;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / nsys;
    const int32_t s = (int32_t)(t - i * nsys);
    out[(int64_t)s * 2 * n + i] = vmid[t];
    out[(int64_t)s * 2 * n + n + i] = vout[t];
  }
}

bool pow2_upto32(int32_t v) { return v == 1 || v == 2 || v == 4 || v == 8 || v == 16 || v == 32; }

void validate_csc(int32_t n, const int32_t* colptr, const int32_t* rowidx) {
  if (n < 0)
    throw InvalidMatrix("negative dimension", -1);
  if (colptr[0] != 0)
    throw InvalidMatrix("colptr[0] != 0", 0);
  for (int32_t j = 0; j < n; ++j) {
    if (colptr[j] > colptr[j + 1])
      throw InvalidMatrix("colptr not non-decreasing", j);
    for (int32_t p = colptr[j]; p < colptr[j + 1]; ++p) {
      if (rowidx[p] < 0 || rowidx[p] >= n)
        throw InvalidMatrix("row index out of range", j);
      if (p > colptr[j] && rowidx[p - 1] >= rowidx[p])
        throw InvalidMatrix("row indices not strictly increasing", j);
    }
  }
}

// Source positions (into M) -> interleaved values of all systems.
void values_from(const DBuf<double>& mval, int64_t nnzM, int32_t nsys, const int32_t* src,
                 int64_t nnz, DBuf<double>& out, cudaStream_t s) {
  out.alloc((nnz > 0 ? nnz : 1) * nsys);
  gather_values(mval.p, nnzM, src, nnz, nsys, out.p, s);
}

void build_plan(sfg_plan* P, const int32_t* colptr, const int32_t* rowidx,
                const double* values, const double* vin_h, uint64_t seed) {
  cudaStream_t s = P->stream;
  const int32_t n = P->n, S = P->nsys;
  const int64_t nnzM = colptr[n];
  P->nnzM = nnzM;
  int64_t lower = 0;
  for (int32_t j = 0; j < n; ++j)
    for (int32_t p = colptr[j]; p < colptr[j + 1]; ++p)
      if (rowidx[p] >= j)
        ++lower;
  P->lower_count = lower;
  if (P->combo == 4) {
    // CSR(A) row r reads x_j for every (r, j) in A: remember the largest j
    P->row_maxcol.assign((size_t)n, -1);
    for (int32_t j = 0; j < n; ++j)
      for (int32_t p = colptr[j]; p < colptr[j + 1]; ++p)
        P->row_maxcol[(size_t)rowidx[p]] = std::max(P->row_maxcol[(size_t)rowidx[p]], j);
  }

  upload(P->m_ptr, colptr, (int64_t)n + 1, s);
  upload(P->m_idx, rowidx, nnzM, s);
  DBuf<double> mval;
  upload(mval, values, nnzM * S, s);

  const int combo = P->combo;
  if (combo == 1 || combo == 2 || combo == 4 || combo == 8 || combo == 5 || combo == 7) {
    // lower_triangle (matrix.hpp:98-128)
    DBuf<int32_t> src;
    P->nnzL = lower_triangle(P->m_ptr.p, P->m_idx.p, mval.p, nnzM, S, n, P->lc_ptr,
                             P->lc_idx, src, s);
    const int64_t nnzL = P->nnzL;
    if (combo == 5 || combo == 7)
      values_from(mval, nnzM, S, src.p, nnzL, P->lc_val, s);
    P->map_lc.alloc(nnzL > 0 ? nnzL : 1);
    SFG_CUDA(cudaMemcpyAsync(P->map_lc.p, src.p, sizeof(int32_t) * (size_t)nnzL,
                             cudaMemcpyDeviceToDevice, s));
    // CSR of L: to_csr (matrix.hpp:66-86), rows ascending columns, diag last
    DBuf<int32_t> csr_ptr((int64_t)n + 1), csr_idx(nnzL > 0 ? nnzL : 1),
        perm(nnzL > 0 ? nnzL : 1), srcc(nnzL > 0 ? nnzL : 1);
    transpose(P->lc_ptr.p, P->lc_idx.p, n, n, nnzL, csr_ptr.p, csr_idx.p, perm.p, s);
    if (combo == 1 || combo == 2 || combo == 4 || combo == 8) {
      compose_kernel<<<grid_for(nnzL), 256, 0, s>>>(src.p, perm.p, nnzL, srcc.p);
      count_launch();
      values_from(mval, nnzM, S, srcc.p, nnzL, P->lr_val, s);
      P->map_lr = std::move(srcc);
      srcc.alloc(nnzL > 0 ? nnzL : 1);
      P->lr_ptr = std::move(csr_ptr);
      P->lr_idx = std::move(csr_idx);
    } else {
      // LowerRowView (kernels.hpp:92-115): perm maps CSR entries to L_csc positions
      P->rv_ptr.alloc((int64_t)n + 1);
      const int64_t nrv = nnzL - n;
      P->rv_col.alloc(nrv > 0 ? nrv : 1);
      P->rv_pos.alloc(nrv > 0 ? nrv : 1);
      rowview_kernel<<<grid_for((int64_t)n + 1), 256, 0, s>>>(csr_ptr.p, csr_idx.p, perm.p, n,
                                                               P->rv_ptr.p, P->rv_col.p,
                                                               P->rv_pos.p);
      count_launch();
    }
    if (combo == 8) {
      // L' rows = L columns reversed: strictly-lower entries by descending
      // row, then the diagonal (the reference's P L^T P^T solve order)
      P->lt_ptr.alloc((int64_t)n + 1);
      SFG_CUDA(cudaMemcpyAsync(P->lt_ptr.p, P->lc_ptr.p, sizeof(int32_t) * ((size_t)n + 1),
                               cudaMemcpyDeviceToDevice, s));
      P->lt_idx.alloc(nnzL > 0 ? nnzL : 1);
      DBuf<int32_t> rperm(nnzL > 0 ? nnzL : 1);
      reverse_segments(P->lc_ptr.p, P->lc_idx.p, n, P->lt_idx.p, rperm.p, s);
      compose_kernel<<<grid_for(nnzL), 256, 0, s>>>(src.p, rperm.p, nnzL, srcc.p);
      count_launch();
      values_from(mval, nnzM, S, srcc.p, nnzL, P->lt_val, s);
      P->map_lt = std::move(srcc);
    }
    if (combo == 2 || combo == 4) {
      // CSR of A: combo 2's SpMV operand (to_csr(M), kernels.hpp:440); for
      // combo 4 the row view of the CSC SpMV operand (row gather, see mline.cu)
      P->ar_ptr.alloc((int64_t)n + 1);
      P->ar_idx.alloc(nnzM > 0 ? nnzM : 1);
      DBuf<int32_t> aperm(nnzM > 0 ? nnzM : 1);
      transpose(P->m_ptr.p, P->m_idx.p, n, n, nnzM, P->ar_ptr.p, P->ar_idx.p, aperm.p, s);
      values_from(mval, nnzM, 1, aperm.p, nnzM, P->ar_val, s);
      P->map_ar = std::move(aperm);
    }
    if (combo == 7) {
      P->dvec.alloc(n > 0 ? n : 1);
      dscal_vector(P->lc_ptr.p, P->lc_val.p, n, P->dvec.p, s);
    }
    if (combo == 4)
      P->m_val = std::move(mval);
    if (combo == 5 || combo == 7) {
      P->nnzF = nnzL;
      P->fac.alloc(nnzL > 0 ? nnzL : 1);
      P->work.alloc(nnzL > 0 ? nnzL : 1);
    }
  } else if (combo == 6 || combo == 3) {
    // to_csr(M) (kernels.hpp:475-478) + find_diag_positions
    P->ar_ptr.alloc((int64_t)n + 1);
    P->ar_idx.alloc(nnzM > 0 ? nnzM : 1);
    DBuf<int32_t> aperm(nnzM > 0 ? nnzM : 1);
    transpose(P->m_ptr.p, P->m_idx.p, n, n, nnzM, P->ar_ptr.p, P->ar_idx.p, aperm.p, s);
    values_from(mval, nnzM, 1, aperm.p, nnzM, P->ar_val, s);
    P->map_ar = std::move(aperm);
    P->diag.alloc(n > 0 ? n : 1);
    find_diag_positions(P->ar_ptr.p, P->ar_idx.p, n, P->diag.p, s);
    if (combo == 3) { // scaling_vector (kernels.hpp:299-309), part of make_state
      P->dvec.alloc(n > 0 ? n : 1);
      const int32_t bad = scaling_vector_csr(P->diag.p, P->ar_val.p, n, P->dvec.p, s);
      if (bad >= 0)
        throw FactorizationFailure("zero diagonal at index " + std::to_string(bad),
                                   SFG_FERR_ZERO_DIAG_SCALE, bad);
    }
    P->nnzF = nnzM;
    P->fac.alloc(nnzM > 0 ? nnzM : 1);
    P->work.alloc(nnzM > 0 ? nnzM : 1);
  }

  // vectors
  const int64_t nv = (int64_t)n * S;
  if (combo != 7 && combo != 3) {
    std::vector<double> hv;
    const double* src_h = vin_h;
    if (!vin_h) {
      hv.resize((size_t)nv);
      for (int32_t sys = 0; sys < S; ++sys)
        sfg_gen_vector(n, seed + (uint64_t)sys, hv.data() + (size_t)sys * n);
      src_h = hv.data();
    }
    P->staging.alloc(nv > 0 ? 2 * nv : 1);
    P->vin.alloc(nv > 0 ? nv : 1);
    if (nv > 0) {
      SFG_CUDA(cudaMemcpyAsync(P->staging.p, src_h, sizeof(double) * (size_t)nv,
                               cudaMemcpyHostToDevice, s));
      interleave(P->staging.p, n, S, P->vin.p, s);
    }
    // one extra all-zero row n: the chain-ELL padding reads it
    P->vout.alloc(nv + S);
    SFG_CUDA(cudaMemsetAsync(P->vout.p + nv, 0, sizeof(double) * (size_t)S, s));
    if (combo == 1 || combo == 2 || combo == 4 || combo == 8) {
      P->vmid.alloc(nv + S);
      SFG_CUDA(cudaMemsetAsync(P->vmid.p + nv, 0, sizeof(double) * (size_t)S, s));
    }
  }
  P->counter.alloc(2); // ticket counter + auxiliary counter
  P->err.alloc(1);
  SFG_CUDA(cudaStreamSynchronize(s));
}

ExecArgs exec_args(sfg_plan* P) {
  ExecArgs a;
  a.n = P->n;
  a.nsys = P->nsys;
  a.order = P->order.p;
  a.counter = P->counter.p;
  a.err = P->err.p;
  a.lr_ptr = P->lr_ptr.p;
  a.lr_idx = P->lr_idx.p;
  a.lr_val = P->lr_val.p;
  a.lt_ptr = P->lt_ptr.p;
  a.lt_idx = P->lt_idx.p;
  a.lt_val = P->lt_val.p;
  a.ar_ptr = P->ar_ptr.p;
  a.ar_idx = P->ar_idx.p;
  a.ar_val = P->ar_val.p;
  a.diag = P->diag.p;
  a.lc_ptr = P->lc_ptr.p;
  a.lc_idx = P->lc_idx.p;
  a.lc_val = P->lc_val.p;
  a.rv_ptr = P->rv_ptr.p;
  a.rv_col = P->rv_col.p;
  a.rv_pos = P->rv_pos.p;
  a.dvec = P->dvec.p;
  a.vin = P->vin.p;
  a.vmid = P->vmid.p;
  a.vout = P->vout.p;
  a.fac = P->fac.p;
  a.work = P->work.p;
  // the warp factorization executors wait on one task per warp: pure spin
  // detects a published word soonest (measured: C4 13.1 -> 11.9 ms vs a
  // 160 ns back-off); the level-set kernels keep the back-off
  if (P->use_warpfac)
    a.sleep_cap = 0;
  if (const char* e = getenv("SFG_SLEEP_CAP"))
    a.sleep_cap = (unsigned)atoi(e);
  if (P->use_warpfac) {
    // resident warps for about `look` levels of claimed tasks and no more:
    // on a DAG of narrow levels the extra warps only spin beside the ones
    // on the critical path (C4, ~110 columns per level: 4 -> 2 blocks/SM,
    // 9.19 -> 8.70 ms); wide-level DAGs (C2, C3) keep full occupancy
    // The same rule sizes the unfused comparator's launches.  Level width is
    // the median over the waves (a few very wide levels beside a long narrow
    // tail do not buy full occupancy; the 90th percentile gave C4 3 blocks/SM,
    // 8.72 -> 8.89 ms).
    int look = 20;
    if (const char* e = getenv("SFG_FACT_LOOKAHEAD"))
      look = std::max(0, std::min(atoi(e), 100000));
    const int64_t waves = std::max<int64_t>(1, (int64_t)P->wave_ptr.size() - 1);
    std::vector<int64_t> width((size_t)waves, 0);
    for (int64_t w = 0; w + 1 < (int64_t)P->wave_ptr.size(); ++w)
      width[(size_t)w] = P->wave_ptr[(size_t)w + 1] - P->wave_ptr[(size_t)w];
    const size_t k50 = (size_t)(0.5 * (double)(waves - 1));
    std::nth_element(width.begin(), width.begin() + k50, width.end());
    const double per_level = (double)std::max<int64_t>(1, width[k50]);
    const double warps = (double)look * per_level;
    if (look > 0)
      a.blocks_per_sm = std::max(
          1, (int)std::min(64.0, std::ceil(warps / ((double)fact_warps_per_block() * sm_count()))));
  }
  if (const char* e = getenv("SFG_BLOCKS_PER_SM"))
    a.blocks_per_sm = atoi(e);
  if (P->use_warpfac && P->trace.p)
    a.ftrace = P->trace.p;
  return a;
}

void ensure_events(sfg_plan* P) {
  for (auto& e : P->ev)
    if (!e)
      SFG_CUDA(cudaEventCreate(&e));
}

// The main executor launch for a ticket range and phase mask.
void launch_main(sfg_plan* P, const ExecArgs& a) {
  switch (P->combo) {
  case 1:
  case 4:
  case 8:
    launch_trsv_pair(P->combo, a, P->stream);
    break;
  case 5:
  case 7:
    if (P->use_warpfac)
      launch_ic0_warp(P->combo, a, P->upd, P->stream);
    else
      launch_ic0(P->combo, a, P->stream);
    break;
  case 3:
  case 6:
    if (P->use_warpfac)
      launch_ilu0_warp(P->combo, a, P->upd, P->stream);
    else
      launch_ilu0(P->combo, a, P->stream);
    break;
  }
}

void do_inspect(sfg_plan* P) {
  if (P->inspected)
    return;
  cudaStream_t s = P->stream;
  const int32_t n = P->n;
  const int combo = P->combo;
  const bool two_segments = combo == 4 || combo == 8;
  P->ntickets = two_segments ? 2 * (int64_t)n : n;
  P->order.alloc(P->ntickets > 0 ? P->ntickets : 1);
  DBuf<int32_t> level(n > 0 ? n : 1);
  const int32_t *ptr = nullptr, *idx = nullptr;
  switch (combo) {
  case 1:
  case 2:
  case 4:
  case 8:
    ptr = P->lr_ptr.p;
    idx = P->lr_idx.p;
    break;
  case 5:
  case 7:
    ptr = P->rv_ptr.p;
    idx = P->rv_col.p;
    break;
  case 3:
  case 6:
    ptr = P->ar_ptr.p;
    idx = P->ar_idx.p;
    break;
  }
  const int32_t P1 = levels_syncfree(ptr, idx, n, +1, level.p, s);
  std::vector<int64_t> w1;
  order_by_level(level.p, n, P1, P->order.p, &w1, s);
  P->wave_ptr = w1;
  P->seg2_start_wave = -1;
  if (combo == 4) {
    iota_i32_kernel<<<grid_for(n), 256, 0, s>>>(P->order.p + n, n, 0);
    count_launch();
    P->seg2_start_wave = (int32_t)P->wave_ptr.size() - 1;
    P->wave_ptr.push_back(2 * (int64_t)n);
  } else if (combo == 8) {
    const int32_t P2 = levels_syncfree(P->lt_ptr.p, P->lt_idx.p, n, -1, level.p, s);
    std::vector<int64_t> w2;
    order_by_level(level.p, n, P2, P->order.p + n, &w2, s);
    P->seg2_start_wave = (int32_t)P->wave_ptr.size() - 1;
    for (size_t k = 1; k < w2.size(); ++k)
      P->wave_ptr.push_back(w2[k] + n);
  }
  const char* ex = getenv("SFG_EXECUTOR");
  const bool legacy = ex && std::string(ex) == "levels";
  // executor choice: the multi-chain warp executor for single-system solve
  // pairs (latency-bound: in-warp dependencies go through shared memory),
  // the chain executor for batched systems; SFG_EXECUTOR overrides
  // single systems: the multi-line executor, except for solve pairs whose L
  // rows carry many dependencies (>= 8 per row on average, e.g. the 27-point
  // grid), where one warp per chain is faster (C5 single system: chain 2.71
  // ms, multi-line 4.89 ms; C1's 5-point rows (3 per row) favour multi-line)
  const bool dense_rows = (combo == 1 || combo == 8) && n > 0 && P->nnzL >= (int64_t)9 * n;
  const bool want_mline =
      (ex ? std::string(ex) == "mline" : (P->nsys == 1 && !dense_rows)) || combo == 2;
  if (want_mline && (combo == 1 || combo == 2 || combo == 4 || combo == 8)) {
    int32_t max_len = 1 << 20;
    if (const char* e = getenv("SFG_CHAIN_MAX"))
      max_len = atoi(e);
    build_mline(P->lr_ptr.p, P->lr_idx.p, n, +1, P->nsys, max_len, P->ml_f, s);
    if (combo == 8)
      build_mline(P->lt_ptr.p, P->lt_idx.p, n, -1, P->nsys, max_len, P->ml_b, s);
    P->use_mline = true;
    const char* se = getenv("SFG_MLINE_STREAM");
    if (P->nsys == 1 && !(se && std::string(se) == "0")) { // step streams (k_mline1)
      build_mline_stream(P->lr_ptr.p, P->lr_val.p, n, +1, P->ml_f, s);
      if (combo == 8)
        build_mline_stream(P->lt_ptr.p, P->lt_val.p, n, -1, P->ml_b, s);
    }
  } else if (combo == 1 || combo == 4 || combo == 8) {
    P->use_chain = !legacy;
  }
  if (P->use_mline) {
    if (getenv("SFG_MLINE_STATS")) {
      for (const MLineLayout* L : {&P->ml_f, &P->ml_b})
        if (L->nchain > 0)
          fprintf(stderr, "mline dir=%d nchain=%d ngroup=%d levels=%d max_steps=%d est_steps=%d width=%d\n",
                  L->dir, L->nchain, L->ngroup, L->nlevels, L->max_steps, L->est_steps, L->CHN);
    }
    if (getenv("SFG_TRACE")) {
      P->trace_tiles = 4;
      const int64_t items = (int64_t)P->ml_f.ngroup + (n + 31) / 32 +
                            (combo == 8 ? P->ml_b.ngroup : P->ml_f.ngroup);
      P->trace.alloc(items * 4);
      SFG_CUDA(cudaMemsetAsync(P->trace.p, 0, sizeof(unsigned long long) * items * 4, s));
    }
  }
  if (!legacy && (combo == 5 || combo == 7)) {
    build_ic0_updates(P->lc_ptr.p, P->lc_idx.p, P->rv_ptr.p, P->rv_col.p, P->rv_pos.p, n,
                      P->nnzF, P->upd, s);
    P->use_warpfac = ic0_warp_fits(P->upd);
  } else if (!legacy && (combo == 6 || combo == 3)) {
    build_ilu0_updates(P->ar_ptr.p, P->ar_idx.p, P->diag.p, n, P->nnzF, P->upd, s);
    P->use_warpfac = ilu0_warp_fits(P->upd);
    // rows of at most 8 / 16 entries: 4 / 2 same-level rows per warp
    const char* pk = getenv("SFG_ILU_PACK");
    if (P->use_warpfac && P->upd.max_updates <= 4 && !(pk && std::string(pk) == "0")) {
      if (P->upd.max_task <= 8 && !(pk && std::string(pk) == "16"))
        build_packs(P->wave_ptr, 8, P->upd);
      else if (P->upd.max_task <= 16)
        build_packs(P->wave_ptr, 16, P->upd);
    }
  }
  if (!P->use_warpfac)
    P->upd = UpdateLists{};
  if (P->use_warpfac && getenv("SFG_TRACE")) {
    P->trace.alloc((int64_t)n * 5);
    SFG_CUDA(cudaMemsetAsync(P->trace.p, 0, sizeof(unsigned long long) * (size_t)n * 5, s));
  }
  if (P->use_chain) {
    if (const char* e = getenv("SFG_CHAIN_G"))
      P->tile_rows = atoi(e);
    const int32_t G = chain_G(P->nsys, P->tile_rows), CS = chain_CS(P->nsys);
    int32_t max_len = 4096;
    if (const char* e = getenv("SFG_CHAIN_MAX"))
      max_len = atoi(e);
    build_chains(P->lr_ptr.p, P->lr_idx.p, n, +1, G, CS, max_len, P->ch_f, s);
    if (combo == 8)
      build_chains(P->lt_ptr.p, P->lt_idx.p, n, -1, G, CS, max_len, P->ch_b, s);
    if (combo == 4)
      build_tails(P->ch_f, P->ar_ptr.p, P->ar_idx.p, n, P->tail_ptr, P->tail_rows, s);
    if (getenv("SFG_TRACE")) {
      P->trace_tiles = getenv("SFG_TRACE_TILES") ? atoi(getenv("SFG_TRACE_TILES")) : 160;
      const int64_t items = (int64_t)P->ch_f.nbatch + P->ch_b.nbatch;
      P->trace.alloc(items * P->trace_tiles * 3);
      SFG_CUDA(cudaMemsetAsync(P->trace.p, 0, sizeof(unsigned long long) * items * P->trace_tiles * 3, s));
      // (the chain-ELL kernel uses one word per tile: the first third)
    }
  }
  SFG_CUDA(cudaStreamSynchronize(s));
  P->inspected = true;
}

MLineArgs mline_args(sfg_plan* P) {
  MLineArgs a;
  a.combo = P->combo;
  a.n = P->n;
  a.S = P->nsys;
  a.counter = P->counter.p;
  a.err = P->err.p;
  a.lr_ptr = P->lr_ptr.p;
  a.lr_idx = P->lr_idx.p;
  a.lr_val = P->lr_val.p;
  a.f_cstart = P->ml_f.cstart.p;
  a.f_cskew = P->ml_f.cskew.p;
  a.f_gsteps = P->ml_f.gsteps.p;
  a.f_gorder = P->ml_f.gorder.p;
  a.f_code = P->ml_f.code.p;
  a.f_nchain = P->ml_f.nchain;
  a.f_ngroup = P->ml_f.ngroup;
  const MLineLayout& L2 = P->combo == 8 ? P->ml_b : P->ml_f;
  a.ar_ptr = P->ar_ptr.p;
  a.ar_idx = P->ar_idx.p;
  a.ar_val = P->ar_val.p;
  a.lt_ptr = P->combo == 8 ? P->lt_ptr.p : P->lr_ptr.p;
  a.lt_idx = P->combo == 8 ? P->lt_idx.p : P->lr_idx.p;
  a.lt_val = P->combo == 8 ? P->lt_val.p : P->lr_val.p;
  a.b_cstart = L2.cstart.p;
  a.b_cskew = L2.cskew.p;
  a.b_gsteps = L2.gsteps.p;
  a.b_gorder = L2.gorder.p;
  a.b_code = L2.code.p;
  a.b_nchain = L2.nchain;
  a.b_ngroup = P->combo == 4 ? (P->n + 31) / 32 : L2.ngroup;
  if (P->combo == 2) { // SpMV row blocks first, then the solve groups
    a.f_ngroup = (P->n + 31) / 32;
    a.b_ngroup = P->ml_f.ngroup;
  }
  a.vin = P->vin.p;
  a.vmid = P->vmid.p;
  a.vout = P->vout.p;
  a.chn = std::max(P->ml_f.CHN, L2.CHN);
  a.trace = P->trace.p;
  a.use_stream = P->ml_f.stream && L2.stream && P->ml_f.sch == L2.sch;
  a.stream_ch = P->ml_f.sch;
  a.f_sofs = P->ml_f.sofs.p;
  a.f_srow = P->ml_f.srow.p;
  a.f_scode = P->ml_f.scode.p;
  a.f_sval = P->ml_f.sval.p;
  a.b_sofs = L2.sofs.p;
  a.b_srow = L2.srow.p;
  a.b_scode = L2.scode.p;
  a.b_sval = L2.sval.p;
  if (const char* e = getenv("SFG_SLEEP_CAP"))
    a.sleep_ns = (unsigned)atoi(e);
  if (const char* e = getenv("SFG_MLINE_DX"))
    a.lookahead = atoi(e);
  if (const char* e = getenv("SFG_BLOCKS_PER_SM"))
    a.blocks_per_sm = atoi(e);
  return a;
}

ChainArgs chain_args(sfg_plan* P) {
  ChainArgs a;
  a.combo = P->combo;
  a.n = P->n;
  a.S = P->nsys;
  a.counter = P->counter.p;
  a.err = P->err.p;
  a.lr_ptr = P->lr_ptr.p;
  a.lr_idx = P->lr_idx.p;
  a.lr_val = P->lr_val.p;
  a.f_cstart = P->ch_f.cstart.p;
  a.f_corder = P->ch_f.corder.p;
  a.f_bptr = P->ch_f.batch_ptr.p;
  a.f_level = P->ch_f.clevel.p;
  a.f_nbatch = P->ch_f.nbatch;
  a.lt_ptr = P->lt_ptr.p;
  a.lt_idx = P->lt_idx.p;
  a.lt_val = P->lt_val.p;
  a.b_cstart = P->ch_b.cstart.p;
  a.b_corder = P->ch_b.corder.p;
  a.b_bptr = P->ch_b.batch_ptr.p;
  a.b_level = P->ch_b.clevel.p;
  a.b_nbatch = P->ch_b.nbatch;
  a.tail_ptr = P->tail_ptr.p;
  a.tile_rows = P->tile_rows;
  if (const char* e = getenv("SFG_CHAIN_SKEW"))
    a.skew_mul = atoi(e);
  a.tail_rows = P->tail_rows.p;
  if (const char* e = getenv("SFG_BWD_GATE"))
    a.bwd_gate = (unsigned)atoi(e);
  a.ar_ptr = P->ar_ptr.p;
  a.ar_idx = P->ar_idx.p;
  a.ar_val = P->ar_val.p;
  a.vin = P->vin.p;
  a.vmid = P->vmid.p;
  a.vout = P->vout.p;
  if (const char* e = getenv("SFG_BLOCKS_PER_SM"))
    a.blocks_per_sm = atoi(e);
  if (P->trace.p) {
    a.trace = P->trace.p;
    a.trace_tiles = P->trace_tiles;
  }
  return a;
}

// ---- parity DAGs ---------------------------------------------------------
void build_cost(sfg_plan* P, int kind, const int32_t* ptr, const int32_t* idx,
                const int32_t* ptr2, const int32_t* aux1, const int32_t* aux2, DevDag& g) {
  g.cost.alloc(P->n > 0 ? P->n : 1);
  if (P->n > 0) {
    cost_kernel<<<grid_for(P->n), 256, 0, P->stream>>>(kind, P->n, ptr, idx, ptr2, aux1, aux2,
                                                       g.cost.p);
    count_launch();
  }
}

void dag_from_structure(sfg_plan* P, const int32_t* ptr, const int32_t* idx, int64_t nent,
                        int mode, DevDag& g) {
  DBuf<uint64_t> keys(nent > 0 ? nent : 1);
  if (nent > 0) {
    edge_keys_kernel<<<grid_for((int64_t)P->n * 32), 256, 0, P->stream>>>(
        ptr, idx, P->n, mode, P->n, 0, 0, keys.p);
    count_launch();
  }
  csr_from_edge_keys(keys, nent, P->n, g, P->stream);
}

void edgeless(sfg_plan* P, DevDag& g) {
  g.nvert = P->n;
  g.nedges = 0;
  g.ptr.alloc((int64_t)P->n + 1);
  SFG_CUDA(cudaMemsetAsync(g.ptr.p, 0, sizeof(int32_t) * ((size_t)P->n + 1), P->stream));
  g.idx.alloc(1);
}

void build_g(sfg_plan* P, int which) {
  auto g = std::make_unique<DevDag>();
  const int c = P->combo;
  const int32_t n = P->n;
  cudaStream_t s = P->stream;
  if (which == 1) { // build_g1 (dag.hpp:319-337)
    if (c == 1 || c == 4 || c == 8) {
      dag_from_structure(P, P->lr_ptr.p, P->lr_idx.p, P->nnzL, EM_ROWS_LOWER, *g);
      build_cost(P, CK_ROWNNZ, P->lr_ptr.p, nullptr, nullptr, nullptr, nullptr, *g);
    } else if (c == 5) {
      dag_from_structure(P, P->lc_ptr.p, P->lc_idx.p, P->nnzL, EM_COLS_BELOW, *g);
      build_cost(P, CK_IC0, P->lc_ptr.p, nullptr, P->rv_ptr.p, P->rv_col.p, P->rv_pos.p, *g);
    } else if (c == 6) {
      dag_from_structure(P, P->ar_ptr.p, P->ar_idx.p, P->nnzM, EM_ROWS_LOWER, *g);
      build_cost(P, CK_ILU0, P->ar_ptr.p, P->ar_idx.p, nullptr, P->diag.p, nullptr, *g);
    } else if (c == 7) {
      edgeless(P, *g);
      build_cost(P, CK_ROWNNZ, P->lc_ptr.p, nullptr, nullptr, nullptr, nullptr, *g);
    } else if (c == 2 || c == 3) { // SpMV_CSR / DSCAL_CSR over A: independent rows
      edgeless(P, *g);
      build_cost(P, CK_ROWNNZ, P->ar_ptr.p, nullptr, nullptr, nullptr, nullptr, *g);
    }
  } else { // build_g2 (dag.hpp:339-370)
    if (c == 1 || c == 2) {
      dag_from_structure(P, P->lr_ptr.p, P->lr_idx.p, P->nnzL, EM_ROWS_LOWER, *g);
      build_cost(P, CK_ROWNNZ, P->lr_ptr.p, nullptr, nullptr, nullptr, nullptr, *g);
    } else if (c == 4) {
      edgeless(P, *g);
      build_cost(P, CK_ROWNNZ, P->m_ptr.p, nullptr, nullptr, nullptr, nullptr, *g);
    } else if (c == 5) {
      dag_from_structure(P, P->lc_ptr.p, P->lc_idx.p, P->nnzL, EM_COLS_BELOW, *g);
      build_cost(P, CK_TRSV_CSC, nullptr, nullptr, P->rv_ptr.p, nullptr, nullptr, *g);
    } else if (c == 6) {
      dag_from_structure(P, P->ar_ptr.p, P->ar_idx.p, P->nnzM, EM_ROWS_LOWER, *g);
      build_cost(P, CK_UNIT, P->ar_ptr.p, P->ar_idx.p, nullptr, nullptr, nullptr, *g);
    } else if (c == 3) { // SpILU0_CSR over A
      dag_from_structure(P, P->ar_ptr.p, P->ar_idx.p, P->nnzM, EM_ROWS_LOWER, *g);
      build_cost(P, CK_ILU0, P->ar_ptr.p, P->ar_idx.p, nullptr, P->diag.p, nullptr, *g);
    } else if (c == 7) {
      dag_from_structure(P, P->lc_ptr.p, P->lc_idx.p, P->nnzL, EM_COLS_BELOW, *g);
      build_cost(P, CK_IC0, P->lc_ptr.p, nullptr, P->rv_ptr.p, P->rv_col.p, P->rv_pos.p, *g);
    } else if (c == 8) {
      dag_from_structure(P, P->lt_ptr.p, P->lt_idx.p, P->nnzL, EM_LT_REV, *g);
      build_cost(P, CK_LT_REV, P->lt_ptr.p, nullptr, nullptr, nullptr, nullptr, *g);
    }
  }
  (void)n;
  SFG_CUDA(cudaStreamSynchronize(s));
  P->dags[which - 1] = std::move(g);
}

void build_fdep(sfg_plan* P) {
  cudaStream_t s = P->stream;
  const int32_t n = P->n;
  auto f = std::make_unique<DevDag>();
  f->nvert = n;
  f->ptr.alloc((int64_t)n + 1);
  DBuf<int32_t> cnt((int64_t)n + 1);
  fdep_count_kernel<<<grid_for((int64_t)n + 1), 256, 0, s>>>(P->combo, n, P->m_ptr.p,
                                                              P->rv_ptr.p, P->ar_ptr.p,
                                                              P->ar_idx.p, cnt.p);
  count_launch();
  size_t bytes = 0;
  SFG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, cnt.p, f->ptr.p, n + 1, s));
  DBuf<char> tmp((int64_t)bytes);
  SFG_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, cnt.p, f->ptr.p, n + 1, s));
  int32_t nnz = 0;
  SFG_CUDA(cudaMemcpyAsync(&nnz, f->ptr.p + n, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  SFG_CUDA(cudaStreamSynchronize(s));
  f->nedges = nnz;
  f->idx.alloc(nnz > 0 ? nnz : 1);
  fdep_fill_kernel<<<grid_for(n), 256, 0, s>>>(P->combo, n, P->m_ptr.p, P->rv_ptr.p,
                                               P->rv_col.p, P->ar_ptr.p, P->ar_idx.p, f->ptr.p,
                                               f->idx.p);
  count_launch();
  SFG_CUDA(cudaStreamSynchronize(s));
  P->fdep = std::move(f);
}

__global__ void cost_concat_kernel(const int64_t* a, const int64_t* b, int32_t n, int64_t* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < 2 * (int64_t)n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = i < n ? a[i] : b[i - n];
}

void build_joint(sfg_plan* P) {
  if (!P->dags[0])
    build_g(P, 1);
  if (!P->dags[1])
    build_g(P, 2);
  if (!P->fdep)
    build_fdep(P);
  const DevDag& g1 = *P->dags[0];
  const DevDag& g2 = *P->dags[1];
  const DevDag& f = *P->fdep;
  cudaStream_t s = P->stream;
  const int32_t n = P->n;
  const int64_t ne = g1.nedges + g2.nedges + f.nedges;
  DBuf<uint64_t> keys(ne > 0 ? ne : 1);
  // joint_dag (dag.hpp:222-238): E1, E2 offset by |V1|, (j, |V1| + i) per F_ij
  if (g1.nedges)
    edge_keys_kernel<<<grid_for((int64_t)n * 32), 256, 0, s>>>(g1.ptr.p, g1.idx.p, n, EM_SUCC,
                                                               n, 0, 0, keys.p);
  if (g2.nedges)
    edge_keys_kernel<<<grid_for((int64_t)n * 32), 256, 0, s>>>(g2.ptr.p, g2.idx.p, n, EM_SUCC,
                                                               n, n, n, keys.p + g1.nedges);
  if (f.nedges)
    edge_keys_kernel<<<grid_for((int64_t)n * 32), 256, 0, s>>>(
        f.ptr.p, f.idx.p, n, EM_FDEP, n, 0, n, keys.p + g1.nedges + g2.nedges);
  count_launch(3);
  auto j = std::make_unique<DevDag>();
  csr_from_edge_keys(keys, ne, 2 * n, *j, s);
  j->cost.alloc(2 * (int64_t)n > 0 ? 2 * (int64_t)n : 1);
  cost_concat_kernel<<<grid_for(2 * (int64_t)n), 256, 0, s>>>(g1.cost.p, g2.cost.p, n, j->cost.p);
  count_launch();
  SFG_CUDA(cudaStreamSynchronize(s));
  P->dags[2] = std::move(j);
}

void ensure_dag(sfg_plan* P, int which) {
  if (which == 3) {
    if (!P->dags[2])
      build_joint(P);
  } else if (!P->dags[which - 1]) {
    build_g(P, which);
  }
}

void ensure_levels(sfg_plan* P, int which) {
  if (P->have_levels[which - 1])
    return;
  ensure_dag(P, which);
  const DevDag& g = *P->dags[which - 1];
  if (!edges_ascend(g, P->stream))
    throw InvalidArgument("dependence cycle: edge does not ascend");
  DevDag pred;
  flip_dag(g, pred, P->stream);
  const int32_t nv = g.nvert;
  P->lev[which - 1].alloc(nv > 0 ? nv : 1);
  P->hgt[which - 1].alloc(nv > 0 ? nv : 1);
  P->slk[which - 1].alloc(nv > 0 ? nv : 1);
  const int32_t Pc = levels_syncfree(pred.ptr.p, pred.idx.p, nv, +1, P->lev[which - 1].p,
                                     P->stream);
  heights_syncfree(g.ptr.p, g.idx.p, nv, P->hgt[which - 1].p, P->stream);
  slack_from(P->lev[which - 1].p, P->hgt[which - 1].p, Pc, nv, P->slk[which - 1].p, P->stream);
  SFG_CUDA(cudaStreamSynchronize(P->stream));
  P->crit[which - 1] = Pc;
  P->have_levels[which - 1] = true;
}

// ---- error word ------------------------------------------------------------
int ferr_kind_of(int combo, int kernel) {
  switch (combo) {
  case 5:
    return kernel == 1 ? SFG_FERR_NONPOS_PIVOT : SFG_FERR_ZERO_DIAG_SOLVE;
  case 3:
  case 6:
    return SFG_FERR_ZERO_PIVOT;
  case 7:
    return SFG_FERR_NONPOS_PIVOT;
  default:
    return SFG_FERR_ZERO_DIAG_SOLVE;
  }
}

const char* ferr_text(int kind) {
  switch (kind) {
  case SFG_FERR_ZERO_DIAG_SOLVE:
    return "zero diagonal in triangular solve";
  case SFG_FERR_NONPOS_PIVOT:
    return "non-positive pivot";
  case SFG_FERR_ZERO_PIVOT:
    return "zero pivot";
  case SFG_FERR_ZERO_DIAG_SCALE:
    return "zero diagonal";
  default:
    return "invalid matrix";
  }
}

sfg_status decode_error_key(sfg_plan* P, unsigned long long key) {
  if (key == ~0ull)
    return SFG_OK;
  const int kernel = (int)(key >> 62) + 1;
  const int32_t index = (int32_t)(key & 0x7fffffffull);
  const int kind = ferr_kind_of(P->combo, kernel);
  return set_err(P, SFG_ERR_FACTORIZATION,
                 std::string(ferr_text(kind)) + " at index " + std::to_string(index), kind,
                 index);
}

sfg_status check_error_word(sfg_plan* P) {
  unsigned long long key = ~0ull;
  SFG_CUDA(cudaMemcpyAsync(&key, P->err.p, sizeof(key), cudaMemcpyDeviceToHost, P->stream));
  SFG_CUDA(cudaStreamSynchronize(P->stream));
  return decode_error_key(P, key);
}

// collect_outputs (kernels.hpp:585-608) of every system into a device buffer
// in the host-facing layout (system-major), on the plan stream.
void collect_to_device(sfg_plan* P, double* dst) {
  const int c = P->combo;
  const int32_t n = P->n, S = P->nsys;
  cudaStream_t s = P->stream;
  if (n == 0)
    return;
  if (c == 1 || c == 2 || c == 4 || c == 8) {
    if (S == 1) {
      SFG_CUDA(cudaMemcpyAsync(dst, P->vmid.p, sizeof(double) * (size_t)n,
                               cudaMemcpyDeviceToDevice, s));
      SFG_CUDA(cudaMemcpyAsync(dst + n, P->vout.p, sizeof(double) * (size_t)n,
                               cudaMemcpyDeviceToDevice, s));
    } else {
      collect_pair_kernel<<<grid_for((int64_t)n * S), 256, 0, s>>>(P->vmid.p, P->vout.p, n, S,
                                                                   dst);
      count_launch();
    }
  } else {
    if (P->nnzF)
      SFG_CUDA(cudaMemcpyAsync(dst, P->fac.p, sizeof(double) * (size_t)P->nnzF,
                               cudaMemcpyDeviceToDevice, s));
    const double* tail = (c == 7 || c == 3) ? P->dvec.p : P->vout.p;
    SFG_CUDA(cudaMemcpyAsync(dst + P->nnzF, tail, sizeof(double) * (size_t)n,
                             cudaMemcpyDeviceToDevice, s));
  }
}

// One fused execution: re-initialise outputs + ticket counter + error word,
// then the single executor launch, bracketed by kb / ke.
void exec_fused_impl(sfg_plan* P, cudaEvent_t kb, cudaEvent_t ke) {
  const int64_t nv = (int64_t)P->n * P->nsys;
  FillRegion r[3];
  int nr = 0;
  // fused fwd -> bwd on the batched chain executor resets vout in-kernel
  // (ChainArgs::bwd_reset): k_prep only resets vmid
  const bool inkernel_reset = P->combo == 8 && P->use_chain && P->nsys >= 2 && P->ch_f.nbatch > 0 &&
                              nv % 2 == 0 && !getenv("SFG_PREP_VOUT");
  switch (P->combo) {
  case 1:
  case 2:
  case 8:
    r[nr++] = {P->vmid.p, nv};
    if (!inkernel_reset)
      r[nr++] = {P->vout.p, nv};
    break;
  case 4:
    r[nr++] = {P->vmid.p, nv};
    break;
  case 5:
  case 6:
    r[nr++] = {P->fac.p, P->nnzF};
    r[nr++] = {P->vout.p, nv};
    break;
  case 3:
  case 7:
    r[nr++] = {P->fac.p, P->nnzF};
    break;
  }
  launch_prep(r, nr, P->counter.p, P->err.p, P->stream);
  SFG_CUDA(cudaEventRecord(kb, P->stream));
  if (P->use_mline) {
    MLineArgs m = mline_args(P);
    m.seg_begin = 0;
    m.seg_end = m.f_ngroup + m.b_ngroup;
    launch_mline(m, P->stream);
  } else if (P->use_chain) {
    ChainArgs b = chain_args(P);
    b.phase = 3;
    if (inkernel_reset) {
      b.bwd_reset = P->vout.p;
      b.bwd_reset_words = nv;
      b.bwd_reset_items = std::min<int32_t>(P->ch_f.nbatch, 512);
      b.reset_done = P->counter.p + 1;
    }
    b.seg_begin = 0;
    b.seg_end = P->ch_f.nbatch + (P->combo == 8 ? P->ch_b.nbatch : 0);
    launch_chain(b, P->stream);
  } else {
    ExecArgs a = exec_args(P);
    a.phase = 3;
    a.t_begin = 0;
    a.t_end = P->ntickets;
    launch_main(P, a);
  }
  SFG_CUDA(cudaEventRecord(ke, P->stream));
}

// Joint-DAG level sets, ascending vertex id within a level
// (build_wavefront_schedule, executor.hpp:209-229), on the GPU: a stable sort
// of the joint vertices by their joint level.
void ensure_wavefront(sfg_plan* P) {
  if (P->have_wf)
    return;
  ensure_levels(P, 3);
  const int32_t nv = 2 * P->n;
  P->wf_verts.alloc(nv > 0 ? nv : 1);
  order_by_level(P->lev[2].p, nv, P->crit[2], P->wf_verts.p, &P->wf_ptr, P->stream);
  P->wf_lptr.alloc((int64_t)P->wf_ptr.size());
  SFG_CUDA(cudaMemcpyAsync(P->wf_lptr.p, P->wf_ptr.data(), sizeof(int64_t) * P->wf_ptr.size(),
                           cudaMemcpyHostToDevice, P->stream));
  SFG_CUDA(cudaStreamSynchronize(P->stream));
  P->have_wf = true;
}

// execute_joint_wavefront (executor.hpp:465-507): the joint level sets one
// after another with a grid barrier between them (wavefront.cu).
void exec_wavefront_impl(sfg_plan* P, cudaEvent_t kb, cudaEvent_t ke) {
  launch_prep(nullptr, 0, P->counter.p, P->err.p, P->stream);
  if (P->combo == 4 && P->n > 0) // spmv_csc_col accumulates into y = 0 (reset, kernels.hpp:498-502)
    SFG_CUDA(cudaMemsetAsync(P->vout.p, 0, sizeof(double) * (size_t)P->n, P->stream));
  SFG_CUDA(cudaEventRecord(kb, P->stream));
  ExecArgs a = exec_args(P);
  launch_wavefront(a, P->combo, P->wf_verts.p, P->wf_lptr.p, (int32_t)P->wf_ptr.size() - 1,
                   P->m_ptr.p, P->m_idx.p, P->m_val.p, P->stream);
  SFG_CUDA(cudaGetLastError());
  SFG_CUDA(cudaEventRecord(ke, P->stream));
}

// execute_sequential (executor.hpp:315-322): run_sequential_reference on one
// GPU thread -- the reference's sequential baseline, same outputs.
void exec_sequential_impl(sfg_plan* P, cudaEvent_t kb, cudaEvent_t ke) {
  launch_prep(nullptr, 0, P->counter.p, P->err.p, P->stream);
  if (P->combo == 4 && P->n > 0)
    SFG_CUDA(cudaMemsetAsync(P->vout.p, 0, sizeof(double) * (size_t)P->n, P->stream));
  SFG_CUDA(cudaEventRecord(kb, P->stream));
  ExecArgs a = exec_args(P);
  launch_wavefront(a, P->combo, nullptr, nullptr, -1, P->m_ptr.p, P->m_idx.p, P->m_val.p,
                   P->stream);
  SFG_CUDA(cudaEventRecord(ke, P->stream));
}

// The unfused comparator (execute_unfused, executor.hpp:325-383): kernel 1
// alone, then kernel 2 alone; stream order is the barrier between them.
// which = 1 / 2 runs only that kernel (sfg_execute_kernel); kernel 2 alone
// reads kernel 1's outputs from the previous call.
void exec_unfused_impl(sfg_plan* P, cudaEvent_t kb, cudaEvent_t ke, int which = 3) {
  const int64_t nv = (int64_t)P->n * P->nsys;
  const int c = P->combo;
  const int32_t n = P->n;
  const bool k1 = which & 1, k2 = which & 2;
  ExecArgs a = exec_args(P);
  FillRegion r1[2];
  int n1 = 0;
  if (c == 1 || c == 2 || c == 4 || c == 8)
    r1[n1++] = {P->vmid.p, nv};
  else if (c == 5 || c == 6)
    r1[n1++] = {P->fac.p, P->nnzF};
  if (k1)
    launch_prep(r1, n1, P->counter.p, P->err.p, P->stream);
  SFG_CUDA(cudaEventRecord(kb, P->stream));
  if (P->use_mline) {
    MLineArgs m = mline_args(P);
    if (k1) {
      m.seg_begin = 0;
      m.seg_end = m.f_ngroup;
      launch_mline(m, P->stream);
    }
    if (k2) {
      FillRegion r2[1] = {{P->vout.p, nv}};
      launch_prep(r2, 1, P->counter.p, nullptr, P->stream);
      m.seg_begin = m.f_ngroup;
      m.seg_end = m.f_ngroup + m.b_ngroup;
      launch_mline(m, P->stream);
    }
    SFG_CUDA(cudaEventRecord(ke, P->stream));
    return;
  }
  if (P->use_chain) {
    ChainArgs b = chain_args(P);
    if (k1) {
      b.phase = 1;
      b.seg_begin = 0;
      b.seg_end = P->ch_f.nbatch;
      launch_chain(b, P->stream);
    }
    if (k2) {
      FillRegion r2[1];
      int n2 = 0;
      if (c == 1 || c == 8)
        r2[n2++] = {P->vout.p, nv};
      launch_prep(r2, n2, P->counter.p, nullptr, P->stream);
      b.phase = 2;
      b.seg_begin = 0;
      b.seg_end = P->ch_f.nbatch;
      if (c == 8) {
        b.seg_begin = P->ch_f.nbatch;
        b.seg_end = P->ch_f.nbatch + P->ch_b.nbatch;
      }
      launch_chain(b, P->stream);
    }
    SFG_CUDA(cudaEventRecord(ke, P->stream));
    return;
  }
  if (k1) {
    a.phase = 1;
    a.t_begin = 0;
    a.t_end = n;
    if (c == 7)
      launch_dscal(a, P->stream);
    else if (c == 3)
      launch_dscal_csr(a, P->stream);
    else
      launch_main(P, a);
  }
  if (k2) {
    FillRegion r2[2];
    int n2 = 0;
    if (c == 1 || c == 8 || c == 5 || c == 6)
      r2[n2++] = {P->vout.p, nv};
    else if (c == 7 || c == 3)
      r2[n2++] = {P->fac.p, P->nnzF};
    launch_prep(r2, n2, P->counter.p, nullptr, P->stream);
    a.phase = 2;
    a.t_begin = 0;
    a.t_end = n;
    if (c == 4 || c == 8) {
      a.t_begin = n;
      a.t_end = 2 * (int64_t)n;
    }
    launch_main(P, a);
  }
  SFG_CUDA(cudaEventRecord(ke, P->stream));
}

__global__ void spmv_rows_kernel(const int32_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                                 const double* __restrict__ val, int32_t r0, int32_t r1,
                                 const double* __restrict__ x, double* __restrict__ y) {
  for (int64_t r = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < r1;
       r += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int32_t p = ptr[r]; p < ptr[r + 1]; ++p)
      acc = __dadd_rn(acc, __dmul_rn(val[p], x[idx[p]]));
    y[r - r0] = acc;
  }
}

} // namespace

// ===========================================================================
extern "C" {

const char* sfg_version(void) { return "sfgpu 0.1 (sm_100a)"; }

sfg_status sfg_set_device(int32_t device) {
  int cnt = 0;
  if (cudaGetDeviceCount(&cnt) != cudaSuccess || cnt <= 0) {
    cudaGetLastError();
    return SFG_ERR_NO_DEVICE;
  }
  if (device < 0 || device >= cnt)
    return SFG_ERR_INVALID_ARGUMENT;
  return cudaSetDevice(device) == cudaSuccess ? SFG_OK : SFG_ERR_CUDA;
}

sfg_status sfg_host_alloc(size_t bytes, void** p) {
  if (!p)
    return SFG_ERR_INVALID_ARGUMENT;
  *p = nullptr;
  int cnt = 0;
  if (cudaGetDeviceCount(&cnt) != cudaSuccess || cnt <= 0) {
    cudaGetLastError();
    return SFG_ERR_NO_DEVICE;
  }
  return cudaHostAlloc(p, bytes > 0 ? bytes : 1, cudaHostAllocDefault) == cudaSuccess
             ? SFG_OK
             : SFG_ERR_CUDA;
}

sfg_status sfg_host_free(void* p) {
  if (p)
    cudaFreeHost(p);
  return SFG_OK;
}

sfg_status sfg_device_check(int32_t* device_count, int32_t* sms) {
  int cnt = 0;
  if (cudaGetDeviceCount(&cnt) != cudaSuccess || cnt <= 0) {
    cudaGetLastError();
    if (device_count)
      *device_count = 0;
    return SFG_ERR_NO_DEVICE;
  }
  if (device_count)
    *device_count = cnt;
  if (sms) {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    *sms = v;
  }
  return SFG_OK;
}

sfg_status sfg_plan_create(int32_t combo, int32_t n, const int32_t* colptr,
                           const int32_t* rowidx, const double* values, int32_t nsys,
                           const double* vin, uint64_t seed, sfg_plan** out) {
  if (!out)
    return SFG_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  if (combo < 1 || combo > 8)
    return SFG_ERR_INVALID_ARGUMENT;
  if (n < 0 || !colptr || (colptr[n] > 0 && (!rowidx || !values)))
    return SFG_ERR_INVALID_ARGUMENT;
  if (nsys < 1 || !pow2_upto32(nsys) || (nsys > 1 && combo != 1 && combo != 8))
    return SFG_ERR_INVALID_ARGUMENT;
  int cnt = 0;
  if (cudaGetDeviceCount(&cnt) != cudaSuccess || cnt <= 0) {
    cudaGetLastError();
    return SFG_ERR_NO_DEVICE;
  }
  auto* P = new sfg_plan();
  P->combo = combo;
  P->n = n;
  P->nsys = nsys;
  cudaGetDevice(&P->device);
  const sfg_status st = guarded(P, [&] {
    validate_csc(n, colptr, rowidx);
    LaunchScope ls(P);
    SFG_CUDA(cudaStreamCreateWithFlags(&P->own_stream, cudaStreamNonBlocking));
    P->stream = P->own_stream;
    build_plan(P, colptr, rowidx, values, vin, seed);
    ensure_events(P);
    return SFG_OK;
  });
  if (st != SFG_OK) {
    // keep the plan alive only to report; callers destroy it on error
    *out = P;
    return st;
  }
  *out = P;
  return SFG_OK;
}

sfg_status sfg_plan_destroy(sfg_plan* P) {
  if (!P)
    return SFG_OK;
  {
    DeviceScope ds(P->device);
    if (P->stream)
      cudaStreamSynchronize(P->stream);
    if (P->trace.p && P->use_warpfac) {
      // SFG_TRACE=<path>: {tasks, 5, 0, data[tasks*5]} (see ExecArgs::ftrace)
      const int64_t items = P->n;
      std::vector<unsigned long long> h((size_t)(items * 5));
      cudaMemcpy(h.data(), P->trace.p, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost);
      if (FILE* f = fopen(getenv("SFG_TRACE"), "wb")) {
        const int64_t hdr[3] = {items, 5, 0};
        fwrite(hdr, sizeof(hdr), 1, f);
        fwrite(h.data(), sizeof(unsigned long long), h.size(), f);
        fclose(f);
      }
    } else if (P->trace.p && P->use_mline) {
      // SFG_TRACE=<path>: {items, 4, fwd items, data[items*4]} (see MLineArgs::trace)
      const int64_t items = (int64_t)P->ml_f.ngroup + (P->combo == 8 ? P->ml_b.ngroup : P->ml_f.ngroup);
      std::vector<unsigned long long> h((size_t)(items * 4));
      cudaMemcpy(h.data(), P->trace.p, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost);
      if (FILE* f = fopen(getenv("SFG_TRACE"), "wb")) {
        const int64_t hdr[3] = {items, 4, P->ml_f.ngroup};
        fwrite(hdr, sizeof(hdr), 1, f);
        fwrite(h.data(), sizeof(unsigned long long), h.size(), f);
        fclose(f);
      }
    } else if (P->trace.p) {
      // SFG_TRACE=<path>: binary dump {items, tiles, data[items*tiles*3]}
      const int64_t items = (int64_t)P->ch_f.nbatch + P->ch_b.nbatch;
      std::vector<unsigned long long> h((size_t)(items * P->trace_tiles * 3));
      cudaMemcpy(h.data(), P->trace.p, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost);
      // chain level of every work item (fwd items then bwd items)
      std::vector<int32_t> lev;
      for (const ChainLayout* L : {&P->ch_f, &P->ch_b}) {
        if (L->nbatch == 0)
          continue;
        std::vector<int32_t> bp((size_t)L->nbatch + 1), co((size_t)L->nchain),
            cl((size_t)L->nchain);
        cudaMemcpy(bp.data(), L->batch_ptr.p, sizeof(int32_t) * bp.size(), cudaMemcpyDeviceToHost);
        cudaMemcpy(co.data(), L->corder.p, sizeof(int32_t) * co.size(), cudaMemcpyDeviceToHost);
        cudaMemcpy(cl.data(), L->clevel.p, sizeof(int32_t) * cl.size(), cudaMemcpyDeviceToHost);
        for (int32_t b = 0; b < L->nbatch; ++b)
          lev.push_back(cl[(size_t)co[(size_t)bp[(size_t)b]]]);
      }
      if (FILE* f = fopen(getenv("SFG_TRACE"), "wb")) {
        const int64_t hdr[3] = {items, P->trace_tiles, P->ch_f.nbatch};
        fwrite(hdr, sizeof(hdr), 1, f);
        fwrite(h.data(), sizeof(unsigned long long), h.size(), f);
        fwrite(lev.data(), sizeof(int32_t), lev.size(), f);
        fclose(f);
      }
    }
    for (auto& e : P->ev)
      if (e)
        cudaEventDestroy(e);
    for (auto& e : P->bev)
      if (e)
        cudaEventDestroy(e);
    if (P->copy_in)
      cudaStreamDestroy(P->copy_in);
    if (P->copy_out)
      cudaStreamDestroy(P->copy_out);
    if (P->own_stream)
      cudaStreamDestroy(P->own_stream);
  }
  delete P;
  return SFG_OK;
}

sfg_status sfg_plan_set_stream(sfg_plan* P, void* stream) {
  if (!P)
    return SFG_ERR_INVALID_ARGUMENT;
  P->stream = stream ? (cudaStream_t)stream : P->own_stream;
  return SFG_OK;
}

sfg_status sfg_plan_info(const sfg_plan* P, int32_t* combo, int32_t* n, int32_t* nsys,
                         int64_t* nnz_factor, int64_t* out_len) {
  if (!P)
    return SFG_ERR_INVALID_ARGUMENT;
  if (combo)
    *combo = P->combo;
  if (n)
    *n = P->n;
  if (nsys)
    *nsys = P->nsys;
  if (nnz_factor)
    *nnz_factor = P->nnzF;
  if (out_len) {
    const int c = P->combo;
    *out_len = (c == 1 || c == 2 || c == 4 || c == 8) ? 2 * (int64_t)P->n : P->nnzF + P->n;
  }
  return SFG_OK;
}

namespace {
sfg_status set_vin_impl(sfg_plan* P, const double* src, cudaMemcpyKind kind) {
  if (!P || !src || P->combo == 7 || P->combo == 3)
    return SFG_ERR_INVALID_ARGUMENT;
  return guarded(P, [&] {
    DeviceScope ds(P->device);
    LaunchScope ls(P);
    const int64_t nv = (int64_t)P->n * P->nsys;
    if (nv == 0)
      return SFG_OK;
    if (P->nsys == 1) {
      SFG_CUDA(cudaMemcpyAsync(P->vin.p, src, sizeof(double) * (size_t)nv, kind, P->stream));
    } else {
      SFG_CUDA(cudaMemcpyAsync(P->staging.p, src, sizeof(double) * (size_t)nv, kind, P->stream));
      interleave(P->staging.p, P->n, P->nsys, P->vin.p, P->stream);
    }
    return SFG_OK;
  });
}
} // namespace

sfg_status sfg_set_vin(sfg_plan* P, const double* vin_host) {
  return set_vin_impl(P, vin_host, cudaMemcpyHostToDevice);
}

sfg_status sfg_set_vin_device(sfg_plan* P, const double* vin_device) {
  return set_vin_impl(P, vin_device, cudaMemcpyDeviceToDevice);
}

namespace {

// Zero diagonal of any system (lower_triangle's check, matrix.hpp:106-112):
// L_csc keeps the diagonal first in every column.
__global__ void diag_check_kernel(const double* __restrict__ mval, int64_t nnzM, int32_t S,
                                  const int32_t* __restrict__ lptr, const int32_t* __restrict__ map,
                                  int32_t n, unsigned long long* bad) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < (int64_t)n * S;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int32_t j = (int32_t)(t / S), sys = (int32_t)(t % S);
    if (mval[(int64_t)sys * nnzM + map[lptr[j]]] == 0.0)
      atomicMin(bad, (unsigned long long)j << 1);
  }
}

} // namespace

sfg_status sfg_set_values(sfg_plan* P, const double* values_host) {
  if (!P || !values_host)
    return SFG_ERR_INVALID_ARGUMENT;
  return guarded(P, [&] {
    DeviceScope ds(P->device);
    LaunchScope ls(P);
    cudaStream_t s = P->stream;
    const int32_t n = P->n, S = P->nsys;
    const int64_t nnzM = P->nnzM, tot = nnzM * S;
    if (tot == 0)
      return SFG_OK;
    if (P->mstage.n < tot)
      P->mstage.alloc(tot);
    SFG_CUDA(cudaMemcpyAsync(P->mstage.p, values_host, sizeof(double) * (size_t)tot,
                             cudaMemcpyHostToDevice, s));
    const int c = P->combo;
    if (c != 6 && c != 3) {
      DBuf<unsigned long long> bad(1);
      SFG_CUDA(cudaMemsetAsync(bad.p, 0xFF, sizeof(unsigned long long), s));
      diag_check_kernel<<<grid_for((int64_t)n * S), 256, 0, s>>>(P->mstage.p, nnzM, S,
                                                                  P->lc_ptr.p, P->map_lc.p, n,
                                                                  bad.p);
      count_launch();
      SFG_CUDA(cudaGetLastError());
      unsigned long long hbad = 0;
      SFG_CUDA(cudaMemcpyAsync(&hbad, bad.p, sizeof(hbad), cudaMemcpyDeviceToHost, s));
      SFG_CUDA(cudaStreamSynchronize(s));
      if (hbad != ~0ull) {
        const int32_t j = (int32_t)(hbad >> 1);
        throw InvalidMatrix("zero diagonal entry at column " + std::to_string(j), j);
      }
    }
    const int64_t nnzL = P->nnzL;
    if (c == 1 || c == 2 || c == 4 || c == 8)
      gather_values(P->mstage.p, nnzM, P->map_lr.p, nnzL, S, P->lr_val.p, s);
    if (c == 8)
      gather_values(P->mstage.p, nnzM, P->map_lt.p, nnzL, S, P->lt_val.p, s);
    if (c == 5 || c == 7)
      gather_values(P->mstage.p, nnzM, P->map_lc.p, nnzL, S, P->lc_val.p, s);
    if (c == 2 || c == 3 || c == 4 || c == 6)
      gather_values(P->mstage.p, nnzM, P->map_ar.p, nnzM, 1, P->ar_val.p, s);
    if (c == 4)
      SFG_CUDA(cudaMemcpyAsync(P->m_val.p, P->mstage.p, sizeof(double) * (size_t)nnzM,
                               cudaMemcpyDeviceToDevice, s));
    if (c == 3) {
      const int32_t bad = scaling_vector_csr(P->diag.p, P->ar_val.p, n, P->dvec.p, s);
      if (bad >= 0)
        throw FactorizationFailure("zero diagonal at index " + std::to_string(bad),
                                   SFG_FERR_ZERO_DIAG_SCALE, bad);
    }
    if (c == 7)
      dscal_vector(P->lc_ptr.p, P->lc_val.p, n, P->dvec.p, s);
    if (P->use_mline && P->ml_f.stream) { // the step streams hold copies of the values
      build_mline_stream(P->lr_ptr.p, P->lr_val.p, n, +1, P->ml_f, s);
      if (c == 8)
        build_mline_stream(P->lt_ptr.p, P->lt_val.p, n, -1, P->ml_b, s);
    }
    SFG_CUDA(cudaGetLastError());
    return SFG_OK;
  });
}

sfg_status sfg_inspect(sfg_plan* P) {
  if (!P)
    return SFG_ERR_INVALID_ARGUMENT;
  return guarded(P, [&] {
    DeviceScope ds(P->device);
    LaunchScope ls(P);
    do_inspect(P);
    return SFG_OK;
  });
}

sfg_status sfg_get_dag(sfg_plan* P, int32_t which, int32_t* nvert, int64_t* nedges,
                       int32_t* succptr, int32_t* succ, int64_t* cost) {
  if (!P || which < 1 || which > 3)
    return SFG_ERR_INVALID_ARGUMENT;
  return guarded(P, [&] {
    DeviceScope ds(P->device);
    LaunchScope ls(P);
    ensure_dag(P, which);
    const DevDag& g = *P->dags[which - 1];
    if (nvert)
      *nvert = g.nvert;
    if (nedges)
      *nedges = g.nedges;
    if (succptr)
      SFG_CUDA(cudaMemcpy(succptr, g.ptr.p, sizeof(int32_t) * ((size_t)g.nvert + 1),
                          cudaMemcpyDeviceToHost));
    if (succ && g.nedges)
      SFG_CUDA(cudaMemcpy(succ, g.idx.p, sizeof(int32_t) * (size_t)g.nedges,
                          cudaMemcpyDeviceToHost));
    if (cost && g.nvert)
      SFG_CUDA(cudaMemcpy(cost, g.cost.p, sizeof(int64_t) * (size_t)g.nvert,
                          cudaMemcpyDeviceToHost));
    return SFG_OK;
  });
}

sfg_status sfg_get_interdep(sfg_plan* P, int32_t* nrows, int32_t* ncols, int64_t* nnz,
                            int32_t* rowptr, int32_t* colidx) {
  if (!P)
    return SFG_ERR_INVALID_ARGUMENT;
  return guarded(P, [&] {
    DeviceScope ds(P->device);
    LaunchScope ls(P);
    if (!P->fdep)
      build_fdep(P);
    const DevDag& f = *P->fdep;
    if (nrows)
      *nrows = P->n;
    if (ncols)
      *ncols = P->n;
    if (nnz)
      *nnz = f.nedges;
    if (rowptr)
      SFG_CUDA(cudaMemcpy(rowptr, f.ptr.p, sizeof(int32_t) * ((size_t)P->n + 1),
                          cudaMemcpyDeviceToHost));
    if (colidx && f.nedges)
      SFG_CUDA(cudaMemcpy(colidx, f.idx.p, sizeof(int32_t) * (size_t)f.nedges,
                          cudaMemcpyDeviceToHost));
    return SFG_OK;
  });
}

sfg_status sfg_get_levels(sfg_plan* P, int32_t which, int32_t* level, int32_t* height,
                          int32_t* slack, int32_t* critical_path) {
  if (!P || which < 1 || which > 3)
    return SFG_ERR_INVALID_ARGUMENT;
  return guarded(P, [&] {
    DeviceScope ds(P->device);
    LaunchScope ls(P);
    ensure_levels(P, which);
    const int32_t nv = P->dags[which - 1]->nvert;
    if (level && nv)
      SFG_CUDA(cudaMemcpy(level, P->lev[which - 1].p, sizeof(int32_t) * (size_t)nv,
                          cudaMemcpyDeviceToHost));
    if (height && nv)
      SFG_CUDA(cudaMemcpy(height, P->hgt[which - 1].p, sizeof(int32_t) * (size_t)nv,
                          cudaMemcpyDeviceToHost));
    if (slack && nv)
      SFG_CUDA(cudaMemcpy(slack, P->slk[which - 1].p, sizeof(int32_t) * (size_t)nv,
                          cudaMemcpyDeviceToHost));
    if (critical_path)
      *critical_path = P->crit[which - 1];
    return SFG_OK;
  });
}

sfg_status sfg_dag_levels(int32_t nvert, const int32_t* succptr, const int32_t* succ,
                          int32_t* level, int32_t* height, int32_t* slack,
                          int32_t* critical_path) {
  if (nvert < 0 || (nvert > 0 && (!succptr || (!succ && succptr[nvert] > 0))))
    return SFG_ERR_INVALID_ARGUMENT;
  try {
    int dc = 0;
    if (cudaGetDeviceCount(&dc) != cudaSuccess || dc == 0)
      return SFG_ERR_NO_DEVICE;
    cudaStream_t s = nullptr;
    DevDag g;
    g.nvert = nvert;
    g.nedges = nvert > 0 ? succptr[nvert] : 0;
    g.ptr.alloc((int64_t)nvert + 1);
    g.idx.alloc(g.nedges > 0 ? g.nedges : 1);
    SFG_CUDA(cudaMemcpy(g.ptr.p, succptr, sizeof(int32_t) * ((size_t)nvert + 1),
                        cudaMemcpyHostToDevice));
    if (g.nedges)
      SFG_CUDA(cudaMemcpy(g.idx.p, succ, sizeof(int32_t) * (size_t)g.nedges,
                          cudaMemcpyHostToDevice));
    if (!edges_ascend(g, s))
      return SFG_ERR_INVALID_ARGUMENT; // "dependence cycle: edge does not ascend"
    DevDag pred;
    flip_dag(g, pred, s);
    DBuf<int32_t> lev(nvert > 0 ? nvert : 1), hgt(nvert > 0 ? nvert : 1), slk(nvert > 0 ? nvert : 1);
    const int32_t Pc = nvert > 0 ? levels_syncfree(pred.ptr.p, pred.idx.p, nvert, +1, lev.p, s) : 0;
    if (nvert > 0) {
      heights_syncfree(g.ptr.p, g.idx.p, nvert, hgt.p, s);
      slack_from(lev.p, hgt.p, Pc, nvert, slk.p, s);
    }
    SFG_CUDA(cudaStreamSynchronize(s));
    if (level && nvert)
      SFG_CUDA(cudaMemcpy(level, lev.p, sizeof(int32_t) * (size_t)nvert, cudaMemcpyDeviceToHost));
    if (height && nvert)
      SFG_CUDA(cudaMemcpy(height, hgt.p, sizeof(int32_t) * (size_t)nvert, cudaMemcpyDeviceToHost));
    if (slack && nvert)
      SFG_CUDA(cudaMemcpy(slack, slk.p, sizeof(int32_t) * (size_t)nvert, cudaMemcpyDeviceToHost));
    if (critical_path)
      *critical_path = Pc;
    return SFG_OK;
  } catch (...) {
    return SFG_ERR_CUDA;
  }
}

sfg_status sfg_compute_reuse(sfg_plan* P, double* reuse) {
  if (!P || !reuse)
    return SFG_ERR_INVALID_ARGUMENT;
  // dag.hpp:374-431 from the nonzero counts
  const double dn = (double)P->n;
  const double L = (double)P->lower_count;
  const double A = (double)P->nnzM;
  switch (P->combo) {
  case 1:
  case 8:
    *reuse = (2 * dn + 2 * L) / std::max(2 * dn + L, L + 2 * dn);
    break;
  case 2:
  case 4:
    *reuse = 2 * dn / std::max(2 * dn + L, A + 2 * dn);
    break;
  case 3:
    *reuse = 2 * A / std::max(A, A + 2 * dn);
    break;
  case 5:
  case 7:
    *reuse = 2 * L / std::max(L, L + 2 * dn);
    break;
  case 6:
    *reuse = 2 * A / std::max(A, L + 2 * dn);
    break;
  default:
    return SFG_ERR_INVALID_ARGUMENT;
  }
  return SFG_OK;
}

sfg_status sfg_get_schedule(sfg_plan* P, int64_t* nentries, uint8_t* tags, int32_t* iters,
                            int32_t* nwaves, int64_t* wave_ptr) {
  if (!P)
    return SFG_ERR_INVALID_ARGUMENT;
  if (!P->inspected)
    return set_err(P, SFG_ERR_LOGIC, "sfg_inspect has not run");
  if (P->use_mline) {
    return guarded(P, [&] {
      DeviceScope ds(P->device);
      auto fetch = [](const DBuf<int32_t>& d, int64_t cnt) {
        std::vector<int32_t> h((size_t)std::max<int64_t>(cnt, 0));
        if (cnt > 0)
          SFG_CUDA(cudaMemcpy(h.data(), d.p, sizeof(int32_t) * (size_t)cnt, cudaMemcpyDeviceToHost));
        return h;
      };
      std::vector<uint8_t> tg;
      std::vector<int32_t> it;
      std::vector<int64_t> wp{0};
      // groups in claim order; inside a group, rows in step order
      auto emit = [&](const MLineLayout& L, uint8_t tag) {
        const auto cs = fetch(L.cstart, (int64_t)L.nchain + 1);
        const auto sk = fetch(L.cskew, L.nchain);
        const auto go = fetch(L.gorder, L.ngroup);
        const auto gs = fetch(L.gsteps, L.ngroup);
        for (int32_t q = 0; q < L.ngroup; ++q) {
          const int32_t g = go[(size_t)q];
          const int32_t c0 = g * L.B, c1 = std::min(L.nchain, c0 + L.B);
          for (int32_t st = 0; st < gs[(size_t)g]; ++st)
            for (int32_t c = c0; c < c1; ++c) {
              const int32_t o = st - sk[(size_t)c];
              if (o >= 0 && o < cs[(size_t)c + 1] - cs[(size_t)c]) {
                tg.push_back(tag);
                it.push_back(cs[(size_t)c] + o); // position (combo 8: i' = n-1-row)
              }
            }
          wp.push_back((int64_t)tg.size());
        }
      };
      if (P->combo == 2) { // SpMV rows first, then the solve groups
        for (int32_t r = 0; r < P->n; ++r) {
          tg.push_back(1);
          it.push_back(r);
          if ((r & 31) == 31 || r == P->n - 1)
            wp.push_back((int64_t)tg.size());
        }
        emit(P->ml_f, 2);
      } else {
        emit(P->ml_f, 1);
      }
      if (P->combo == 2) {
      } else if (P->combo == 4) { // SpMV rows after every forward row
        for (int32_t r = 0; r < P->n; ++r) {
          tg.push_back(2);
          it.push_back(r);
          if ((r & 31) == 31 || r == P->n - 1)
            wp.push_back((int64_t)tg.size());
        }
      } else {
        emit(P->combo == 8 ? P->ml_b : P->ml_f, 2);
      }
      if (nentries)
        *nentries = (int64_t)tg.size();
      if (nwaves)
        *nwaves = (int32_t)wp.size() - 1;
      if (wave_ptr)
        std::copy(wp.begin(), wp.end(), wave_ptr);
      if (tags)
        std::copy(tg.begin(), tg.end(), tags);
      if (iters)
        std::copy(it.begin(), it.end(), iters);
      return SFG_OK;
    });
  }
  if (P->use_chain) {
    return guarded(P, [&] {
      DeviceScope ds(P->device);
      const int32_t n = P->n;
      auto fetch = [](const DBuf<int32_t>& d, int64_t cnt) {
        std::vector<int32_t> h((size_t)std::max<int64_t>(cnt, 0));
        if (cnt > 0)
          SFG_CUDA(cudaMemcpy(h.data(), d.p, sizeof(int32_t) * (size_t)cnt, cudaMemcpyDeviceToHost));
        return h;
      };
      std::vector<uint8_t> tg;
      std::vector<int32_t> it;
      std::vector<int64_t> wp{0};
      auto emit = [&](const ChainLayout& L, bool bwd) {
        const auto cs = fetch(L.cstart, (int64_t)L.nchain + 1);
        const auto co = fetch(L.corder, L.nchain);
        const auto bp = fetch(L.batch_ptr, (int64_t)L.nbatch + 1);
        std::vector<int32_t> tp, tr;
        if (P->combo == 4 && !bwd) {
          tp = fetch(P->tail_ptr, (int64_t)L.nchain + 1);
          tr = fetch(P->tail_rows, n);
        }
        for (int32_t bi = 0; bi < L.nbatch; ++bi) {
          for (int32_t q = bp[(size_t)bi]; q < bp[(size_t)bi + 1]; ++q) {
            const int32_t c = co[(size_t)q];
            for (int32_t p = cs[(size_t)c]; p < cs[(size_t)c + 1]; ++p) {
              if (bwd) {
                tg.push_back(2);
                it.push_back(p); // reversed numbering i' = n-1-row = position
              } else {
                tg.push_back(1);
                it.push_back(p);
                if (P->combo == 1) {
                  tg.push_back(2);
                  it.push_back(p);
                }
              }
            }
          }
          if (!tp.empty())
            for (int32_t q = bp[(size_t)bi]; q < bp[(size_t)bi + 1]; ++q) {
              const int32_t c = co[(size_t)q];
              for (int32_t t = tp[(size_t)c]; t < tp[(size_t)c + 1]; ++t) {
                tg.push_back(2);
                it.push_back(tr[(size_t)t]);
              }
            }
          wp.push_back((int64_t)tg.size());
        }
      };
      emit(P->ch_f, false);
      if (P->combo == 8)
        emit(P->ch_b, true);
      if (nentries)
        *nentries = (int64_t)tg.size();
      if (nwaves)
        *nwaves = (int32_t)wp.size() - 1;
      if (wave_ptr)
        std::copy(wp.begin(), wp.end(), wave_ptr);
      if (tags)
        std::copy(tg.begin(), tg.end(), tags);
      if (iters)
        std::copy(it.begin(), it.end(), iters);
      return SFG_OK;
    });
  }
  return guarded(P, [&] {
    DeviceScope ds(P->device);
    const bool fused_task = !(P->combo == 4 || P->combo == 8);
    const int64_t ne = fused_task ? 2 * P->ntickets : P->ntickets;
    if (nentries)
      *nentries = ne;
    if (nwaves)
      *nwaves = (int32_t)P->wave_ptr.size() - 1;
    if (wave_ptr) {
      for (size_t k = 0; k < P->wave_ptr.size(); ++k)
        wave_ptr[k] = fused_task ? 2 * P->wave_ptr[k] : P->wave_ptr[k];
    }
    if (tags || iters) {
      std::vector<int32_t> ord((size_t)P->ntickets);
      if (P->ntickets)
        SFG_CUDA(cudaMemcpy(ord.data(), P->order.p, sizeof(int32_t) * ord.size(),
                            cudaMemcpyDeviceToHost));
      for (int64_t t = 0; t < P->ntickets; ++t) {
        if (fused_task) {
          if (tags) {
            tags[2 * t] = 1;
            tags[2 * t + 1] = 2;
          }
          if (iters) {
            iters[2 * t] = ord[(size_t)t];
            iters[2 * t + 1] = ord[(size_t)t];
          }
        } else {
          if (tags)
            tags[t] = t < P->n ? 1 : 2;
          if (iters)
            iters[t] = (P->combo == 8 && t >= P->n) ? P->n - 1 - ord[(size_t)t]
                                                    : ord[(size_t)t];
        }
      }
    }
    return SFG_OK;
  });
}

namespace {

// The executor's schedule as the reference's FusedPartitioning (msp.hpp:44-63):
// s-partitions run one after another, their w-partitions are independent and
// each w-partition is an ordered list of (kernel, iteration) entries.  Every
// executor here orders its work by a dependency level (chain-DAG or group-DAG
// level for the solve executors, task level for the others), so the levels
// are the s-partitions and the sequential work units -- a chain, a group in
// step order, a fused task, a block of SpMV rows -- the w-partitions.
struct Partition {
  std::vector<int64_t> s_ptr{0}, w_ptr{0};
  std::vector<uint8_t> tags;
  std::vector<int32_t> iters;
  void entry(uint8_t t, int32_t i) {
    tags.push_back(t);
    iters.push_back(i);
  }
  void end_w() { w_ptr.push_back((int64_t)tags.size()); }
  void end_s() {
    if ((int64_t)w_ptr.size() - 1 > s_ptr.back())
      s_ptr.push_back((int64_t)w_ptr.size() - 1);
  }
};

std::vector<int32_t> fetch_i32(const DBuf<int32_t>& d, int64_t cnt) {
  std::vector<int32_t> h((size_t)std::max<int64_t>(cnt, 0));
  if (cnt > 0)
    SFG_CUDA(cudaMemcpy(h.data(), d.p, sizeof(int32_t) * (size_t)cnt, cudaMemcpyDeviceToHost));
  return h;
}

void spmv_blocks(Partition& V, int32_t n, uint8_t tag) {
  for (int32_t r0 = 0; r0 < n; r0 += 32) {
    for (int32_t r = r0; r < std::min(n, r0 + 32); ++r)
      V.entry(tag, r);
    V.end_w();
  }
  V.end_s();
}

void mline_groups(Partition& V, const MLineLayout& L, uint8_t tag) {
  const auto lev = fetch_i32(L.glevel, L.ngroup);
  const auto go = fetch_i32(L.gorder, L.ngroup);
  const auto gs = fetch_i32(L.gsteps, L.ngroup);
  const auto cs = fetch_i32(L.cstart, (int64_t)L.nchain + 1);
  const auto sk = fetch_i32(L.cskew, L.nchain);
  int32_t cur = -1;
  for (int32_t q = 0; q < L.ngroup; ++q) {
    const int32_t g = go[(size_t)q];
    if (lev[(size_t)g] != cur) {
      V.end_s();
      cur = lev[(size_t)g];
    }
    const int32_t c0 = g * L.B, c1 = std::min(L.nchain, c0 + L.B);
    for (int32_t st = 0; st < gs[(size_t)g]; ++st)
      for (int32_t c = c0; c < c1; ++c) {
        const int32_t o = st - sk[(size_t)c];
        if (o >= 0 && o < cs[(size_t)c + 1] - cs[(size_t)c])
          V.entry(tag, cs[(size_t)c] + o);
      }
    V.end_w();
  }
  V.end_s();
}

void chain_levels(Partition& V, const ChainLayout& L, uint8_t tag, bool with_second) {
  const auto lev = fetch_i32(L.clevel, L.nchain);
  const auto co = fetch_i32(L.corder, L.nchain);
  const auto cs = fetch_i32(L.cstart, (int64_t)L.nchain + 1);
  int32_t cur = -1;
  for (int32_t q = 0; q < L.nchain; ++q) {
    const int32_t c = co[(size_t)q];
    if (lev[(size_t)c] != cur) {
      V.end_s();
      cur = lev[(size_t)c];
    }
    for (int32_t p = cs[(size_t)c]; p < cs[(size_t)c + 1]; ++p) {
      V.entry(tag, p);
      if (with_second)
        V.entry(2, p);
    }
    V.end_w();
  }
  V.end_s();
}

void build_partition(sfg_plan* P, Partition& V) {
  const int c = P->combo;
  const int32_t n = P->n;
  if (P->use_mline) {
    if (c == 2) {
      spmv_blocks(V, n, 1);
      mline_groups(V, P->ml_f, 2);
    } else {
      mline_groups(V, P->ml_f, 1);
      if (c == 4)
        spmv_blocks(V, n, 2);
      else
        mline_groups(V, c == 8 ? P->ml_b : P->ml_f, 2);
    }
    return;
  }
  if (P->use_chain) {
    chain_levels(V, P->ch_f, 1, c == 1);
    if (c == 8)
      chain_levels(V, P->ch_b, 2, false);
    else if (c == 4)
      spmv_blocks(V, n, 2);
    return;
  }
  // ticket executors: one s-partition per wavefront, one task per w-partition
  const bool fused_task = !(c == 4 || c == 8);
  const auto ord = fetch_i32(P->order, P->ntickets);
  for (size_t w = 0; w + 1 < P->wave_ptr.size(); ++w) {
    for (int64_t t = P->wave_ptr[w]; t < P->wave_ptr[w + 1]; ++t) {
      const int32_t r = ord[(size_t)t];
      if (fused_task) {
        V.entry(1, r);
        V.entry(2, r);
      } else if (t < n) {
        V.entry(1, r);
      } else {
        V.entry(2, c == 8 ? n - 1 - r : r);
      }
      V.end_w();
    }
    V.end_s();
  }
}

} // namespace

sfg_status sfg_get_partitioning(sfg_plan* P, int32_t* nspart, int64_t* nwpart,
                                int64_t* nentries, int64_t* s_ptr, int64_t* w_ptr,
                                uint8_t* tags, int32_t* iters) {
  if (!P)
    return SFG_ERR_INVALID_ARGUMENT;
  if (!P->inspected)
    return set_err(P, SFG_ERR_LOGIC, "sfg_inspect has not run");
  return guarded(P, [&] {
    DeviceScope ds(P->device);
    Partition V;
    build_partition(P, V);
    if (nspart)
      *nspart = (int32_t)V.s_ptr.size() - 1;
    if (nwpart)
      *nwpart = (int64_t)V.w_ptr.size() - 1;
    if (nentries)
      *nentries = (int64_t)V.tags.size();
    if (s_ptr)
      std::copy(V.s_ptr.begin(), V.s_ptr.end(), s_ptr);
    if (w_ptr)
      std::copy(V.w_ptr.begin(), V.w_ptr.end(), w_ptr);
    if (tags)
      std::copy(V.tags.begin(), V.tags.end(), tags);
    if (iters)
      std::copy(V.iters.begin(), V.iters.end(), iters);
    return SFG_OK;
  });
}

// K executions with new right-hand sides, transfers overlapped with compute:
// the input of step k+1 streams in (copy engine 1) and the outputs of step
// k-1 stream out (copy engine 2) while step k runs.  Each step's error word
// is kept, so a breakdown in any step is reported like sfg_synchronize would.
sfg_status sfg_execute_batch(sfg_plan* P, int32_t nsteps, const double* const* vin_host,
                             double* const* out_host) {
  return sfg_execute_batch_ex(P, nsteps, vin_host, out_host, SFG_OUTPUTS_ALL);
}

sfg_status sfg_execute_batch_ex(sfg_plan* P, int32_t nsteps, const double* const* vin_host,
                                double* const* out_host, int32_t outputs) {
  if (!P || nsteps < 0 || (nsteps > 0 && (!vin_host || !out_host)) || P->combo == 3 ||
      P->combo == 7 || (outputs != SFG_OUTPUTS_ALL && outputs != SFG_OUTPUTS_FINAL))
    return SFG_ERR_INVALID_ARGUMENT;
  if (!P->inspected)
    return set_err(P, SFG_ERR_LOGIC, "sfg_inspect has not run");
  return guarded(P, [&] {
    DeviceScope ds(P->device);
    LaunchScope ls(P);
    if (nsteps == 0)
      return SFG_OK;
    const int32_t n = P->n, S = P->nsys;
    const int64_t nv = (int64_t)n * S;
    const int c = P->combo;
    const bool final_only = outputs == SFG_OUTPUTS_FINAL;
    const int64_t olen =
        final_only ? nv : ((c == 1 || c == 2 || c == 4 || c == 8) ? 2 * (int64_t)n : P->nnzF + n) * S;
    if (!P->copy_in) {
      SFG_CUDA(cudaStreamCreateWithFlags(&P->copy_in, cudaStreamNonBlocking));
      SFG_CUDA(cudaStreamCreateWithFlags(&P->copy_out, cudaStreamNonBlocking));
      for (auto& e : P->bev)
        SFG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    for (int b = 0; b < 2; ++b) {
      if (P->in_stage[b].n < nv)
        P->in_stage[b].alloc(std::max<int64_t>(nv, 1));
      if (P->out_stage[b].n < olen)
        P->out_stage[b].alloc(std::max<int64_t>(olen, 1));
    }
    if (P->err_hist.n < nsteps)
      P->err_hist.alloc(nsteps);
    cudaEvent_t* in_ready = P->bev;      // [2]
    cudaEvent_t* in_free = P->bev + 2;   // [2]
    cudaEvent_t* out_ready = P->bev + 4; // [2]
    cudaEvent_t* out_free = P->bev + 6;  // [2]
    // start with every staging buffer free
    for (int b = 0; b < 2; ++b) {
      SFG_CUDA(cudaEventRecord(in_free[b], P->stream));
      SFG_CUDA(cudaEventRecord(out_free[b], P->stream));
    }
    auto stage_in = [&](int32_t k) {
      const int b = k & 1;
      SFG_CUDA(cudaStreamWaitEvent(P->copy_in, in_free[b], 0));
      SFG_CUDA(cudaMemcpyAsync(P->in_stage[b].p, vin_host[k], sizeof(double) * (size_t)nv,
                               cudaMemcpyHostToDevice, P->copy_in));
      SFG_CUDA(cudaEventRecord(in_ready[b], P->copy_in));
    };
    stage_in(0);
    for (int32_t k = 0; k < nsteps; ++k) {
      const int b = k & 1;
      if (k + 1 < nsteps)
        stage_in(k + 1);
      SFG_CUDA(cudaStreamWaitEvent(P->stream, in_ready[b], 0));
      interleave(P->in_stage[b].p, n, S, P->vin.p, P->stream);
      SFG_CUDA(cudaEventRecord(in_free[b], P->stream));
      exec_fused_impl(P, P->ev[1], P->ev[2]);
      SFG_CUDA(cudaMemcpyAsync(P->err_hist.p + k, P->err.p, sizeof(unsigned long long),
                               cudaMemcpyDeviceToDevice, P->stream));
      SFG_CUDA(cudaStreamWaitEvent(P->stream, out_free[b], 0));
      if (final_only)
        deinterleave(P->vout.p, n, S, P->out_stage[b].p, P->stream);
      else
        collect_to_device(P, P->out_stage[b].p);
      SFG_CUDA(cudaEventRecord(out_ready[b], P->stream));
      SFG_CUDA(cudaStreamWaitEvent(P->copy_out, out_ready[b], 0));
      SFG_CUDA(cudaMemcpyAsync(out_host[k], P->out_stage[b].p, sizeof(double) * (size_t)olen,
                               cudaMemcpyDeviceToHost, P->copy_out));
      SFG_CUDA(cudaEventRecord(out_free[b], P->copy_out));
    }
    SFG_CUDA(cudaStreamSynchronize(P->copy_out));
    SFG_CUDA(cudaStreamSynchronize(P->stream));
    std::vector<unsigned long long> eh((size_t)nsteps);
    SFG_CUDA(cudaMemcpy(eh.data(), P->err_hist.p, sizeof(unsigned long long) * eh.size(),
                        cudaMemcpyDeviceToHost));
    for (unsigned long long key : eh)
      if (key != ~0ull)
        return decode_error_key(P, key);
    P->timed = false;
    return SFG_OK;
  });
}

sfg_status sfg_execute_fused(sfg_plan* P) {
  if (!P)
    return SFG_ERR_INVALID_ARGUMENT;
  if (!P->inspected)
    return set_err(P, SFG_ERR_LOGIC, "sfg_inspect has not run");
  return guarded(P, [&] {
    DeviceScope ds(P->device);
    LaunchScope ls(P);
    SFG_CUDA(cudaEventRecord(P->ev[0], P->stream));
    exec_fused_impl(P, P->ev[1], P->ev[2]);
    SFG_CUDA(cudaEventRecord(P->ev[3], P->stream));
    P->timed = true;
    return SFG_OK;
  });
}

sfg_status sfg_execute_unfused(sfg_plan* P) {
  if (!P)
    return SFG_ERR_INVALID_ARGUMENT;
  if (!P->inspected)
    return set_err(P, SFG_ERR_LOGIC, "sfg_inspect has not run");
  return guarded(P, [&] {
    DeviceScope ds(P->device);
    LaunchScope ls(P);
    SFG_CUDA(cudaEventRecord(P->ev[0], P->stream));
    exec_unfused_impl(P, P->ev[1], P->ev[2]);
    SFG_CUDA(cudaEventRecord(P->ev[3], P->stream));
    P->timed = true;
    return SFG_OK;
  });
}

sfg_status sfg_execute_wavefront(sfg_plan* P) {
  if (!P)
    return SFG_ERR_INVALID_ARGUMENT;
  return guarded(P, [&] {
    DeviceScope ds(P->device);
    LaunchScope ls(P);
    ensure_wavefront(P);
    SFG_CUDA(cudaEventRecord(P->ev[0], P->stream));
    exec_wavefront_impl(P, P->ev[1], P->ev[2]);
    SFG_CUDA(cudaEventRecord(P->ev[3], P->stream));
    P->timed = true;
    return SFG_OK;
  });
}

sfg_status sfg_execute_sequential(sfg_plan* P) {
  if (!P)
    return SFG_ERR_INVALID_ARGUMENT;
  return guarded(P, [&] {
    DeviceScope ds(P->device);
    LaunchScope ls(P);
    SFG_CUDA(cudaEventRecord(P->ev[0], P->stream));
    exec_sequential_impl(P, P->ev[1], P->ev[2]);
    SFG_CUDA(cudaEventRecord(P->ev[3], P->stream));
    P->timed = true;
    return SFG_OK;
  });
}

sfg_status sfg_check_schedule(sfg_plan* P, int64_t nentries, const uint8_t* tags,
                              const int32_t* iters, int64_t* violations) {
  if (!P || !violations || nentries < 0 || (nentries > 0 && (!tags || !iters)))
    return SFG_ERR_INVALID_ARGUMENT;
  return guarded(P, [&] {
    DeviceScope ds(P->device);
    LaunchScope ls(P);
    ensure_dag(P, 3);
    const DevDag& j = *P->dags[2];
    *violations = check_schedule_order(j.ptr.p, j.idx.p, P->n, tags, iters, nentries, P->stream);
    return SFG_OK;
  });
}

sfg_status sfg_get_wavefront(sfg_plan* P, int64_t* nentries, uint8_t* tags, int32_t* iters,
                             int32_t* nlevels, int64_t* level_ptr) {
  if (!P)
    return SFG_ERR_INVALID_ARGUMENT;
  return guarded(P, [&] {
    DeviceScope ds(P->device);
    LaunchScope ls(P);
    ensure_wavefront(P);
    const int32_t n = P->n;
    if (nentries)
      *nentries = 2 * (int64_t)n;
    if (nlevels)
      *nlevels = (int32_t)P->wf_ptr.size() - 1;
    if (level_ptr)
      std::copy(P->wf_ptr.begin(), P->wf_ptr.end(), level_ptr);
    if ((tags || iters) && n > 0) {
      std::vector<int32_t> v((size_t)2 * n);
      SFG_CUDA(cudaMemcpy(v.data(), P->wf_verts.p, sizeof(int32_t) * v.size(),
                          cudaMemcpyDeviceToHost));
      for (size_t q = 0; q < v.size(); ++q) {
        if (tags)
          tags[q] = v[q] < n ? 1 : 2;
        if (iters)
          iters[q] = v[q] < n ? v[q] : v[q] - n;
      }
    }
    return SFG_OK;
  });
}

sfg_status sfg_execute_kernel(sfg_plan* P, int32_t which) {
  if (!P || (which != 1 && which != 2))
    return SFG_ERR_INVALID_ARGUMENT;
  if (!P->inspected)
    return set_err(P, SFG_ERR_LOGIC, "sfg_inspect has not run");
  return guarded(P, [&] {
    DeviceScope ds(P->device);
    LaunchScope ls(P);
    SFG_CUDA(cudaEventRecord(P->ev[0], P->stream));
    exec_unfused_impl(P, P->ev[1], P->ev[2], which);
    SFG_CUDA(cudaEventRecord(P->ev[3], P->stream));
    P->timed = true;
    return SFG_OK;
  });
}

sfg_status sfg_spmv_rows(sfg_plan* P, int32_t r0, int32_t r1, const double* x_device,
                         double* y_device) {
  if (!P || !x_device || !y_device || r0 < 0 || r1 < r0 || r1 > P->n || P->ar_ptr.p == nullptr ||
      P->nsys != 1)
    return SFG_ERR_INVALID_ARGUMENT;
  return guarded(P, [&] {
    DeviceScope ds(P->device);
    LaunchScope ls(P);
    if (r1 > r0) {
      spmv_rows_kernel<<<grid_for(r1 - r0), 256, 0, P->stream>>>(P->ar_ptr.p, P->ar_idx.p,
                                                                 P->ar_val.p, r0, r1, x_device,
                                                                 y_device);
      count_launch();
      SFG_CUDA(cudaGetLastError());
    }
    return SFG_OK;
  });
}

sfg_status sfg_synchronize(sfg_plan* P) {
  if (!P)
    return SFG_ERR_INVALID_ARGUMENT;
  return guarded(P, [&] {
    DeviceScope ds(P->device);
    SFG_CUDA(cudaStreamSynchronize(P->stream));
    return check_error_word(P);
  });
}

sfg_status sfg_reset(sfg_plan* P) {
  if (!P)
    return SFG_ERR_INVALID_ARGUMENT;
  return guarded(P, [&] {
    DeviceScope ds(P->device);
    cudaStream_t s = P->stream;
    const int64_t nv = (int64_t)P->n * P->nsys;
    const int c = P->combo;
    // reset (kernels.hpp:498-502): fac = fac0, vmid = vout = 0
    if (P->nnzF > 0) {
      const double* fac0 = (c == 5 || c == 7) ? P->lc_val.p : P->ar_val.p;
      SFG_CUDA(cudaMemcpyAsync(P->fac.p, fac0, sizeof(double) * (size_t)P->nnzF,
                               cudaMemcpyDeviceToDevice, s));
    }
    if (nv > 0 && P->vmid.p)
      SFG_CUDA(cudaMemsetAsync(P->vmid.p, 0, sizeof(double) * (size_t)nv, s));
    if (nv > 0 && P->vout.p)
      SFG_CUDA(cudaMemsetAsync(P->vout.p, 0, sizeof(double) * (size_t)nv, s));
    SFG_CUDA(cudaStreamSynchronize(s));
    return SFG_OK;
  });
}

sfg_status sfg_collect_outputs(sfg_plan* P, double* out, int64_t cap) {
  if (!P || (!out && cap > 0))
    return SFG_ERR_INVALID_ARGUMENT;
  return guarded(P, [&] {
    DeviceScope ds(P->device);
    LaunchScope ls(P);
    const sfg_status e = check_error_word(P);
    if (e != SFG_OK)
      return e;
    const int c = P->combo;
    const int32_t n = P->n, S = P->nsys;
    cudaStream_t s = P->stream;
    if (c == 1 || c == 2 || c == 4 || c == 8) {
      const int64_t need = 2 * (int64_t)n * S;
      if (cap < need)
        throw InvalidArgument("output buffer too small");
      if (n == 0)
        return SFG_OK;
      if (S == 1) {
        SFG_CUDA(cudaMemcpyAsync(out, P->vmid.p, sizeof(double) * (size_t)n,
                                 cudaMemcpyDeviceToHost, s));
        SFG_CUDA(cudaMemcpyAsync(out + n, P->vout.p, sizeof(double) * (size_t)n,
                                 cudaMemcpyDeviceToHost, s));
      } else {
        collect_pair_kernel<<<grid_for((int64_t)n * S), 256, 0, s>>>(P->vmid.p, P->vout.p, n, S,
                                                                     P->staging.p);
        count_launch();
        SFG_CUDA(cudaMemcpyAsync(out, P->staging.p, sizeof(double) * (size_t)need,
                                 cudaMemcpyDeviceToHost, s));
      }
    } else {
      const int64_t need = P->nnzF + n;
      if (cap < need)
        throw InvalidArgument("output buffer too small");
      if (P->nnzF)
        SFG_CUDA(cudaMemcpyAsync(out, P->fac.p, sizeof(double) * (size_t)P->nnzF,
                                 cudaMemcpyDeviceToHost, s));
      const double* tail = (c == 7 || c == 3) ? P->dvec.p : P->vout.p;
      if (n)
        SFG_CUDA(cudaMemcpyAsync(out + P->nnzF, tail, sizeof(double) * (size_t)n,
                                 cudaMemcpyDeviceToHost, s));
    }
    SFG_CUDA(cudaStreamSynchronize(s));
    return SFG_OK;
  });
}

sfg_status sfg_device_output(sfg_plan* P, int32_t which, void** dptr, int64_t* count) {
  if (!P || !dptr)
    return SFG_ERR_INVALID_ARGUMENT;
  const int c = P->combo;
  const int64_t nv = (int64_t)P->n * P->nsys;
  if (c == 1 || c == 2 || c == 4 || c == 8) {
    *dptr = which == 0 ? (void*)P->vmid.p : (void*)P->vout.p;
    if (count)
      *count = nv;
  } else {
    if (which == 0) {
      *dptr = P->fac.p;
      if (count)
        *count = P->nnzF;
    } else {
      *dptr = (c == 7 || c == 3) ? (void*)P->dvec.p : (void*)P->vout.p;
      if (count)
        *count = P->n;
    }
  }
  return SFG_OK;
}

sfg_status sfg_last_error(const sfg_plan* P, int32_t* kind, int32_t* index, char* msg,
                          int32_t msg_len) {
  if (!P)
    return SFG_ERR_INVALID_ARGUMENT;
  if (kind)
    *kind = P->ferr_kind;
  if (index)
    *index = P->ferr_index;
  if (msg && msg_len > 0) {
    const size_t k = std::min<size_t>(P->msg.size(), (size_t)msg_len - 1);
    std::memcpy(msg, P->msg.data(), k);
    msg[k] = 0;
  }
  return SFG_OK;
}

int64_t sfg_launch_count(const sfg_plan* P) { return P ? P->launches : -1; }

sfg_status sfg_bench_executions(sfg_plan* P, int32_t reps, int32_t unfused, float* total_ms,
                                float* kernel_ms_avg) {
  if (!P || reps < 1)
    return SFG_ERR_INVALID_ARGUMENT;
  if (!P->inspected)
    return set_err(P, SFG_ERR_LOGIC, "sfg_inspect has not run");
  return guarded(P, [&] {
    DeviceScope ds(P->device);
    LaunchScope ls(P);
    if (unfused == 2)
      ensure_wavefront(P);
    std::vector<cudaEvent_t> ev((size_t)2 * reps + 2, nullptr);
    for (auto& e : ev)
      SFG_CUDA(cudaEventCreate(&e));
    SFG_CUDA(cudaEventRecord(ev[0], P->stream));
    for (int r = 0; r < reps; ++r) {
      if (unfused == 2)
        exec_wavefront_impl(P, ev[(size_t)2 + 2 * r], ev[(size_t)3 + 2 * r]);
      else if (unfused)
        exec_unfused_impl(P, ev[(size_t)2 + 2 * r], ev[(size_t)3 + 2 * r]);
      else
        exec_fused_impl(P, ev[(size_t)2 + 2 * r], ev[(size_t)3 + 2 * r]);
    }
    SFG_CUDA(cudaEventRecord(ev[1], P->stream));
    SFG_CUDA(cudaEventSynchronize(ev[1]));
    float tot = 0.f, ksum = 0.f;
    SFG_CUDA(cudaEventElapsedTime(&tot, ev[0], ev[1]));
    for (int r = 0; r < reps; ++r) {
      float ms = 0.f;
      SFG_CUDA(cudaEventElapsedTime(&ms, ev[(size_t)2 + 2 * r], ev[(size_t)3 + 2 * r]));
      ksum += ms;
    }
    for (auto& e : ev)
      cudaEventDestroy(e);
    if (total_ms)
      *total_ms = tot;
    if (kernel_ms_avg)
      *kernel_ms_avg = ksum / (float)reps;
    return check_error_word(P);
  });
}

sfg_status sfg_last_exec_ms(sfg_plan* P, float* total_ms, float* kernel_ms) {
  if (!P || !P->timed)
    return SFG_ERR_INVALID_ARGUMENT;
  return guarded(P, [&] {
    DeviceScope ds(P->device);
    SFG_CUDA(cudaEventSynchronize(P->ev[3]));
    if (total_ms)
      SFG_CUDA(cudaEventElapsedTime(total_ms, P->ev[0], P->ev[3]));
    if (kernel_ms)
      SFG_CUDA(cudaEventElapsedTime(kernel_ms, P->ev[1], P->ev[2]));
    return SFG_OK;
  });
}

} // extern "C"
