// executor.cu -- the fused kernel-pair executor (replaces execute_fused,
// executor.hpp:395-461, and the per-iteration bodies of kernels.hpp:145-286).
//
// One launch runs BOTH kernels of a pair.  Work is claimed as tickets in the
// inspector's dependency order (a wavefront-grouped linear extension of the
// joint DAG); a fused task computes the kernel-1 iteration and the dependent
// kernel-2 iteration back to back, so the shared operand (vector entry or
// factor column) is consumed from registers instead of a round trip through
// HBM, and there is no barrier anywhere: each dependency is one polled word.
//
// Arithmetic follows the reference bit for bit: every accumulation runs in
// the reference's storage order with separately rounded multiply and
// subtract (__dmul_rn / __dsub_rn, no FMA), IEEE division and square root.
#include "common.cuh"
#include "executor.cuh"
#include "internal.hpp"

namespace sfg {

namespace {

constexpr int kBlock = 256;
constexpr int CH = 8;    // nonzeros staged in registers per batch
constexpr int MAXC = 32; // column/row length kept in thread-local arrays

__device__ __forceinline__ double as_f64(unsigned long long b) {
  return __longlong_as_double((long long)b);
}

__device__ __forceinline__ double fsub_mul(double acc, double a, double b) {
  return __dsub_rn(acc, __dmul_rn(a, b));
}

// ---------------------------------------------------------------------------
// Triangular-solve rows (S systems interleaved; lane handles one system).
// ---------------------------------------------------------------------------

// x_r = (rhs - sum_{p<diag} v_p * x[col_p]) / v_diag over CSR row r with the
// diagonal stored last (trsv_csr_row, kernels.hpp:171-181).  The row's
// indices and values are staged in registers, all x loads are issued before
// the first one is consumed, and only words still SENT are re-polled.
template <int S>
__device__ __forceinline__ double solve_row(int r, int s,
                                            const int32_t* __restrict__ ptr,
                                            const int32_t* __restrict__ idx,
                                            const double* __restrict__ val,
                                            double rhs, const double* x,
                                            unsigned long long* err, int kernel,
                                            int seqpos, unsigned cap) {
  const int b = __ldg(ptr + r);
  const int e = __ldg(ptr + r + 1) - 1;
  const double d = __ldg(val + (size_t)e * S + s);
  double acc = rhs;
  for (int p = b; p < e; p += CH) {
    const int cnt = min(CH, e - p);
    int jj[CH];
    double vv[CH];
    unsigned long long xx[CH];
#pragma unroll
    for (int a = 0; a < CH; ++a)
      if (a < cnt) {
        jj[a] = __ldg(idx + p + a);
        vv[a] = __ldg(val + (size_t)(p + a) * S + s);
      }
#pragma unroll
    for (int a = 0; a < CH; ++a)
      if (a < cnt)
        xx[a] = ld_relaxed_u64(x + (size_t)jj[a] * S + s);
#pragma unroll
    for (int a = 0; a < CH; ++a)
      if (a < cnt) {
        const double xj = xx[a] != SENT ? as_f64(xx[a])
                                        : poll_f64(x + (size_t)jj[a] * S + s, cap);
        acc = fsub_mul(acc, vv[a], xj);
      }
  }
  if (d == 0.0)
    report_error(err, kernel, seqpos, r);
  return __ddiv_rn(acc, d);
}

// y_r = sum_p a_p * x[col_p] starting from 0.0 in ascending column order.
// This row gather over CSR(A) adds the terms of y_r in exactly the order the
// sequential CSC scatter (spmv_csc_col, kernels.hpp:162-168, j ascending)
// does, so the result is the sequential reference's bit for bit -- without
// the reference's atomic fetch_add.
__device__ __forceinline__ double gather_row(int r,
                                             const int32_t* __restrict__ ptr,
                                             const int32_t* __restrict__ idx,
                                             const double* __restrict__ val,
                                             const double* x, unsigned cap) {
  const int b = __ldg(ptr + r);
  const int e = __ldg(ptr + r + 1);
  double acc = 0.0;
  for (int p = b; p < e; p += CH) {
    const int cnt = min(CH, e - p);
    int jj[CH];
    double vv[CH];
    unsigned long long xx[CH];
#pragma unroll
    for (int a = 0; a < CH; ++a)
      if (a < cnt) {
        jj[a] = __ldg(idx + p + a);
        vv[a] = __ldg(val + p + a);
      }
#pragma unroll
    for (int a = 0; a < CH; ++a)
      if (a < cnt)
        xx[a] = ld_relaxed_u64(x + jj[a]);
#pragma unroll
    for (int a = 0; a < CH; ++a)
      if (a < cnt) {
        const double xj = xx[a] != SENT ? as_f64(xx[a]) : poll_f64(x + jj[a], cap);
        acc = __dadd_rn(acc, __dmul_rn(vv[a], xj));
      }
  }
  return acc;
}

// Combos 1 (fwd -> fwd), 4 (fwd -> SpMV) and 8 (fwd -> bwd).
//   combo 1: ticket t < n is the fused task r = order[t]: z_r then x2_r
//            (interleaved packing; the second solve's row r only needs z_r
//            and x2 of rows finished earlier).
//   combo 4: t < n forward row order[t]; t >= n SpMV row order[t].
//   combo 8: t < n forward row; t >= n backward row (L' rows, descending
//            wavefronts).
template <int COMBO, int S>
__global__ void __launch_bounds__(kBlock, 2) k_trsv_pair(const ExecArgs A) {
  constexpr int R = 32 / S; // rows per warp claim
  const int lane = threadIdx.x & 31;
  const int slot = lane / S;
  const int s = lane % S;
  const int64_t total = A.t_end - A.t_begin;
  for (;;) {
    const long long base = claim_tickets(A.counter, R);
    if (base >= total)
      break;
    const long long c = base + slot;
    if (c >= total)
      continue;
    const int64_t t = A.t_begin + c;
    const int r = __ldg(A.order + t);
    if (COMBO == 1) {
      double z;
      if (A.phase & 1) {
        z = solve_row<S>(r, s, A.lr_ptr, A.lr_idx, A.lr_val,
                         __ldg(A.vin + (size_t)r * S + s), A.vmid, A.err, 1, r, A.sleep_cap);
        publish_f64(A.vmid + (size_t)r * S + s, z);
      } else {
        z = poll_f64(A.vmid + (size_t)r * S + s, A.sleep_cap);
      }
      if (A.phase & 2) {
        const double x2 = solve_row<S>(r, s, A.lr_ptr, A.lr_idx, A.lr_val, z,
                                       A.vout, A.err, 2, r, A.sleep_cap);
        publish_f64(A.vout + (size_t)r * S + s, x2);
      }
    } else if (t < A.n) { // forward row of kernel 1 (combos 4, 8)
      const double z =
          solve_row<S>(r, s, A.lr_ptr, A.lr_idx, A.lr_val,
                       __ldg(A.vin + (size_t)r * S + s), A.vmid, A.err, 1, r, A.sleep_cap);
      publish_f64(A.vmid + (size_t)r * S + s, z);
    } else if (COMBO == 4) {
      A.vout[r] = gather_row(r, A.ar_ptr, A.ar_idx, A.ar_val, A.vmid, A.sleep_cap);
    } else { // COMBO 8 backward row r of L': rhs z_r, then x_j for j > r
      const double z = poll_f64(A.vmid + (size_t)r * S + s, A.sleep_cap);
      const double x = solve_row<S>(r, s, A.lt_ptr, A.lt_idx, A.lt_val, z,
                                    A.vout, A.err, 2, A.n - 1 - r, A.sleep_cap);
      publish_f64(A.vout + (size_t)r * S + s, x);
    }
  }
}

// ---------------------------------------------------------------------------
// Left-looking IC0 column (ic0_column, kernels.hpp:214-242) fused with the
// CSC-row solve (trsv_csc_row, kernels.hpp:200-210) for combo 5, or with the
// DSCAL scaling applied on load (dscal_csc_col, kernels.hpp:281-286) for
// combo 7.  One thread per column k.
//   src 0: column k from lc_val; 1: scaled on load; 2: pre-scaled in work.
// The reference's dense marker array becomes a merge of two sorted row lists
// (column k and the tail of column j from L(k,j) on, whose start is exactly
// the row view's position -- lower_bound(k) in column j).
// ---------------------------------------------------------------------------
template <int COMBO>
__global__ void __launch_bounds__(kBlock) k_ic0(const ExecArgs A) {
  const int lane = threadIdx.x & 31;
  const int64_t total = A.t_end - A.t_begin;
  const bool do_fac = COMBO == 5 ? (A.phase & 1) : (A.phase & 2);
  const bool do_solve = COMBO == 5 && (A.phase & 2);
  const int src = COMBO == 5 ? 0 : ((A.phase & 1) ? 1 : 2);
  const int fac_kernel = COMBO == 5 ? 1 : 2;
  double accl[MAXC];
  int rowl[MAXC];
  for (;;) {
    const long long base = claim_tickets(A.counter, 32);
    if (base >= total)
      break;
    const long long c = base + lane;
    if (c >= total)
      continue;
    const int k = __ldg(A.order + A.t_begin + c);
    const int c0 = __ldg(A.lc_ptr + k);
    const int c1 = __ldg(A.lc_ptr + k + 1);
    const int m = c1 - c0;
    const int q0 = __ldg(A.rv_ptr + k);
    const int q1 = __ldg(A.rv_ptr + k + 1);
    double acc2 = do_solve ? __ldg(A.vin + k) : 0.0;
    if (do_fac) {
      const bool local = m <= MAXC;
      double* acc = local ? accl : A.work + c0;
      const double dk = src == 1 ? __ldg(A.dvec + k) : 0.0;
      for (int a = 0; a < m; ++a) {
        const int row = __ldg(A.lc_idx + c0 + a);
        if (local)
          rowl[a] = row;
        double v;
        if (src == 0)
          v = __ldg(A.lc_val + c0 + a);
        else if (src == 1)
          v = __dmul_rn(__dmul_rn(__ldg(A.dvec + row), __ldg(A.lc_val + c0 + a)), dk);
        else
          v = A.work[c0 + a];
        acc[a] = v;
      }
      for (int q = q0; q < q1; ++q) {
        const int j = __ldg(A.rv_col + q);
        const int pj = __ldg(A.rv_pos + q);
        const int pe = __ldg(A.lc_ptr + j + 1);
        const double lkj = poll_f64(A.fac + pj, A.sleep_cap);
        if (do_solve)
          acc2 = fsub_mul(acc2, lkj, poll_f64(A.vout + j, A.sleep_cap));
        // merge rows of column j from row k on with the rows of column k
        int a = 0;
        for (int p = pj; p < pe; ++p) {
          const int i = __ldg(A.lc_idx + p);
          while (a < m && (local ? rowl[a] : __ldg(A.lc_idx + c0 + a)) < i)
            ++a;
          if (a == m)
            break;
          if ((local ? rowl[a] : __ldg(A.lc_idx + c0 + a)) == i)
            acc[a] = fsub_mul(acc[a], lkj, poll_f64(A.fac + p, A.sleep_cap));
        }
      }
      const double d = acc[0];
      if (d <= 0.0)
        report_error(A.err, fac_kernel, k, k);
      const double lkk = __dsqrt_rn(d);
      for (int a = 1; a < m; ++a)
        publish_f64(A.fac + c0 + a, __ddiv_rn(acc[a], lkk));
      publish_f64(A.fac + c0, lkk);
      if (do_solve) {
        if (lkk == 0.0)
          report_error(A.err, 2, k, k);
        publish_f64(A.vout + k, __ddiv_rn(acc2, lkk));
      }
    } else if (do_solve) { // combo 5 kernel 2 alone (unfused second launch)
      for (int q = q0; q < q1; ++q)
        acc2 = fsub_mul(acc2, poll_f64(A.fac + __ldg(A.rv_pos + q), A.sleep_cap),
                        poll_f64(A.vout + __ldg(A.rv_col + q), A.sleep_cap));
      const double d = poll_f64(A.fac + c0, A.sleep_cap);
      if (d == 0.0)
        report_error(A.err, 2, k, k);
      publish_f64(A.vout + k, __ddiv_rn(acc2, d));
    }
  }
}

// ---------------------------------------------------------------------------
// IKJ ILU0 row (ilu0_row, kernels.hpp:246-272) fused with the unit-lower
// solve (trsv_csr_unit_row, kernels.hpp:184-196): the solve's l_ik are the
// multipliers the factorization just produced, still in registers.
// ---------------------------------------------------------------------------
// COMBO 3 (DSCAL -> ILU0, kernels.hpp:274-279 then 246-272): the row is
// scaled on load, (d_i * a_ij) * d_j, when fused, or read from `work` after a
// separate DSCAL launch; there is no solve.
template <int COMBO>
__global__ void __launch_bounds__(kBlock) k_ilu0(const ExecArgs A) {
  const int lane = threadIdx.x & 31;
  const int64_t total = A.t_end - A.t_begin;
  const bool do_fac = COMBO == 6 ? (A.phase & 1) : (A.phase & 2);
  const bool do_solve = COMBO == 6 && (A.phase & 2);
  const int src = COMBO == 6 ? 0 : ((A.phase & 1) ? 1 : 2);
  const int fac_kernel = COMBO == 6 ? 1 : 2;
  double accl[MAXC];
  int coll[MAXC];
  for (;;) {
    const long long base = claim_tickets(A.counter, 32);
    if (base >= total)
      break;
    const long long c = base + lane;
    if (c >= total)
      continue;
    const int i = __ldg(A.order + A.t_begin + c);
    const int r0 = __ldg(A.ar_ptr + i);
    const int r1 = __ldg(A.ar_ptr + i + 1);
    const int m = r1 - r0;
    double acc2 = do_solve ? __ldg(A.vin + i) : 0.0;
    if (do_fac) {
      const bool local = m <= MAXC;
      double* acc = local ? accl : A.work + r0;
      const double di = src == 1 ? __ldg(A.dvec + i) : 0.0;
      for (int a = 0; a < m; ++a) {
        const int cj = __ldg(A.ar_idx + r0 + a);
        if (local)
          coll[a] = cj;
        acc[a] = src == 0   ? __ldg(A.ar_val + r0 + a)
                 : src == 1 ? __dmul_rn(__dmul_rn(di, __ldg(A.ar_val + r0 + a)), __ldg(A.dvec + cj))
                            : A.work[r0 + a];
      }
#define COL(a) (local ? coll[(a)] : __ldg(A.ar_idx + r0 + (a)))
      for (int a = 0; a < m; ++a) {
        const int k = COL(a);
        if (k >= i)
          break;
        const int dk = __ldg(A.diag + k);
        const double piv = dk >= 0 ? poll_f64(A.fac + dk, A.sleep_cap) : 0.0;
        if (dk < 0 || piv == 0.0)
          report_error(A.err, fac_kernel, i, k);
        const double lik = __ddiv_rn(acc[a], piv);
        acc[a] = lik;
        if (dk >= 0) {
          const int qe = __ldg(A.ar_ptr + k + 1);
          int b = a + 1;
          for (int q = dk + 1; q < qe; ++q) {
            const int j = __ldg(A.ar_idx + q);
            while (b < m && COL(b) < j)
              ++b;
            if (b == m)
              break;
            if (COL(b) == j)
              acc[b] = fsub_mul(acc[b], lik, poll_f64(A.fac + q, A.sleep_cap));
          }
        }
        if (do_solve)
          acc2 = fsub_mul(acc2, lik, poll_f64(A.vout + k, A.sleep_cap));
      }
#undef COL
      for (int a = 0; a < m; ++a)
        publish_f64(A.fac + r0 + a, acc[a]);
    } else if (do_solve) { // unit solve alone (unfused second launch)
      for (int p = r0; p < r1; ++p) {
        const int k = __ldg(A.ar_idx + p);
        if (k >= i)
          break;
        acc2 = fsub_mul(acc2, poll_f64(A.fac + p, A.sleep_cap), poll_f64(A.vout + k, A.sleep_cap));
      }
    }
    if (do_solve)
      publish_f64(A.vout + i, acc2);
  }
}

// DSCAL over CSR rows alone (combo 3 kernel 1 in the unfused comparator):
// work[p] = (d_i * a_p) * d_j (dscal_csr_row, kernels.hpp:274-279).
__global__ void __launch_bounds__(kBlock) k_dscal_csr(const ExecArgs A) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < A.n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double di = __ldg(A.dvec + i);
    for (int p = __ldg(A.ar_ptr + i); p < __ldg(A.ar_ptr + i + 1); ++p)
      A.work[p] = __dmul_rn(__dmul_rn(di, __ldg(A.ar_val + p)), __ldg(A.dvec + __ldg(A.ar_idx + p)));
  }
}

// DSCAL alone (combo 7 kernel 1 in the unfused comparator).
__global__ void __launch_bounds__(kBlock) k_dscal(const ExecArgs A) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < A.n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const double dk = __ldg(A.dvec + k);
    for (int p = __ldg(A.lc_ptr + k); p < __ldg(A.lc_ptr + k + 1); ++p)
      A.work[p] =
          __dmul_rn(__dmul_rn(__ldg(A.dvec + __ldg(A.lc_idx + p)), __ldg(A.lc_val + p)), dk);
  }
}

struct PrepArgs {
  FillRegion r[3];
  int nregions;
  unsigned long long* counter;
  unsigned long long* err;
};

__global__ void k_prep(const PrepArgs P) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (tid == 0) {
    P.counter[0] = 0ull;
    P.counter[1] = 0ull; // auxiliary counter (chain.cu: backward reset slices)
    if (P.err)
      *P.err = ~0ull;
  }
  for (int k = 0; k < P.nregions; ++k) {
    ulonglong2* p2 = reinterpret_cast<ulonglong2*>(P.r[k].ptr);
    const int64_t n2 = P.r[k].words / 2;
    const ulonglong2 v = make_ulonglong2(SENT, SENT);
    for (int64_t i = tid; i < n2; i += stride)
      p2[i] = v;
    if ((P.r[k].words & 1) && tid == 0)
      reinterpret_cast<unsigned long long*>(P.r[k].ptr)[P.r[k].words - 1] = SENT;
  }
}

template <typename K> int resident_grid(K kernel) {
  int per_sm = 0;
  SFG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kBlock, 0));
  if (per_sm < 1)
    per_sm = 1;
  return per_sm * sm_count();
}

template <typename K> void launch_persistent(K kernel, const ExecArgs& a, cudaStream_t s,
                                             int tickets_per_warp) {
  const int64_t total = a.t_end - a.t_begin;
  if (total <= 0)
    return;
  const int64_t warps_needed = (total + tickets_per_warp - 1) / tickets_per_warp;
  int64_t blocks = (warps_needed + (kBlock / 32) - 1) / (kBlock / 32);
  int64_t cap = resident_grid(kernel);
  if (a.blocks_per_sm > 0 && (int64_t)a.blocks_per_sm * sm_count() < cap)
    cap = (int64_t)a.blocks_per_sm * sm_count();
  if (blocks > cap)
    blocks = cap;
  kernel<<<(unsigned)blocks, kBlock, 0, s>>>(a);
  count_launch();
  SFG_CUDA(cudaGetLastError());
}

template <int COMBO> void launch_trsv_pair_c(const ExecArgs& a, cudaStream_t s) {
  switch (a.nsys) {
  case 1:
    launch_persistent(k_trsv_pair<COMBO, 1>, a, s, 32);
    break;
  case 2:
    launch_persistent(k_trsv_pair<COMBO, 2>, a, s, 16);
    break;
  case 4:
    launch_persistent(k_trsv_pair<COMBO, 4>, a, s, 8);
    break;
  case 8:
    launch_persistent(k_trsv_pair<COMBO, 8>, a, s, 4);
    break;
  case 16:
    launch_persistent(k_trsv_pair<COMBO, 16>, a, s, 2);
    break;
  case 32:
    launch_persistent(k_trsv_pair<COMBO, 32>, a, s, 1);
    break;
  default:
    throw InvalidArgument("nsys must be a power of two <= 32");
  }
}

} // namespace

void launch_prep(const FillRegion* regions, int nregions,
                 unsigned long long* counter, unsigned long long* err,
                 cudaStream_t s) {
  PrepArgs P{};
  P.nregions = nregions;
  int64_t words = 1;
  for (int k = 0; k < nregions; ++k) {
    P.r[k] = regions[k];
    words = words > regions[k].words ? words : regions[k].words;
  }
  P.counter = counter;
  P.err = err;
  int64_t blocks = (words / 2 + kBlock - 1) / kBlock;
  const int64_t cap = (int64_t)sm_count() * 8;
  if (blocks > cap)
    blocks = cap;
  if (blocks < 1)
    blocks = 1;
  k_prep<<<(unsigned)blocks, kBlock, 0, s>>>(P);
  count_launch();
  SFG_CUDA(cudaGetLastError());
}

void launch_trsv_pair(int combo, const ExecArgs& a, cudaStream_t s) {
  if (combo == 1)
    launch_trsv_pair_c<1>(a, s);
  else if (combo == 4) {
    if (a.nsys != 1)
      throw InvalidArgument("combo 4 supports a single system");
    launch_persistent(k_trsv_pair<4, 1>, a, s, 32);
  } else if (combo == 8)
    launch_trsv_pair_c<8>(a, s);
  else
    throw InvalidArgument("launch_trsv_pair: bad combo");
}

void launch_ic0(int combo, const ExecArgs& a, cudaStream_t s) {
  if (combo == 5)
    launch_persistent(k_ic0<5>, a, s, 32);
  else
    launch_persistent(k_ic0<7>, a, s, 32);
}

void launch_ilu0(int combo, const ExecArgs& a, cudaStream_t s) {
  if (combo == 3)
    launch_persistent(k_ilu0<3>, a, s, 32);
  else
    launch_persistent(k_ilu0<6>, a, s, 32);
}

void launch_dscal_csr(const ExecArgs& a, cudaStream_t s) {
  int64_t blocks = ((int64_t)a.n + kBlock - 1) / kBlock;
  const int64_t cap = (int64_t)sm_count() * 8;
  if (blocks > cap)
    blocks = cap;
  if (blocks < 1)
    blocks = 1;
  k_dscal_csr<<<(unsigned)blocks, kBlock, 0, s>>>(a);
  count_launch();
  SFG_CUDA(cudaGetLastError());
}

void launch_dscal(const ExecArgs& a, cudaStream_t s) {
  int64_t blocks = ((int64_t)a.n + kBlock - 1) / kBlock;
  const int64_t cap = (int64_t)sm_count() * 8;
  if (blocks > cap)
    blocks = cap;
  if (blocks < 1)
    blocks = 1;
  k_dscal<<<(unsigned)blocks, kBlock, 0, s>>>(a);
  count_launch();
  SFG_CUDA(cudaGetLastError());
}

} // namespace sfg
