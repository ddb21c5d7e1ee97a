// fact.cu -- update-list inspector and warp-per-task executors for the
// factorization pairs (combos 5, 6, 7).  See fact.cuh for the design.
//
// Arithmetic is the reference's bit for bit: every factor entry receives its
// updates in the reference's order (predecessor column j ascending for IC0,
// kernels.hpp:224-236; pivot k ascending for ILU0, kernels.hpp:253-268) with
// separately rounded multiply and subtract, IEEE square root, and divisions
// that are IEEE-exact (div_with_rcp falls back to the IEEE division outside
// its proven range).
#include <cstdlib>

#include <cub/cub.cuh>

#include "common.cuh"
#include "fact.cuh"

#ifndef SFG_FACT_TRACE
// 1: the warp executors record their task timeline when SFG_TRACE is set
// (diagnostic builds: scripts/build_alt.sh trace "-DSFG_FACT_TRACE=1")
#define SFG_FACT_TRACE 0
#endif

#ifndef SFG_IC_BUNROLL
#define SFG_IC_BUNROLL 0 // unroll factor of the IC0 update-batch loop (2: C4 9.19 -> 9.63 ms)
#endif
#ifndef SFG_IC_UNROLL
#define SFG_IC_UNROLL 2 // unroll factor of the IC0 solve-row loop (C2 0.368 -> 0.362 ms)
#endif
#ifndef SFG_ILU_UNROLL
#define SFG_ILU_UNROLL 2 // unroll factor of the ILU0 pivot-step loop (C3 1.438 -> 1.123 ms; 3: 1.159, 4: 1.438)
#endif

#ifndef SFG_IC5_CHU
// IC0 combo 5: update slots per batch.  Four (72 registers, 3 blocks per SM)
// instead of eight (116 registers, 2 blocks): C2 0.478 -> 0.444 ms; three
// slots compiled for 4 blocks per SM: 0.358 -> 0.348 ms (two: 0.378 ms)
#define SFG_IC5_CHU 3
#endif
#ifndef SFG_IC7_CHU
#define SFG_IC7_CHU 4 // IC0 combo 7: update slots per batch (8: 9.53 ms, 4: 9.18 ms on C4)
#endif
#ifndef SFG_IC7_MINB
#define SFG_IC7_MINB 1 // blocks per SM k_ic0_warp<7> is compiled for (A/B builds)
#endif
#ifndef SFG_IC5_MINB
#define SFG_IC5_MINB 4 // blocks per SM k_ic0_warp<5> is compiled for (A/B builds)
#endif

#ifndef SFG_ILU_MINB4
#define SFG_ILU_MINB4 3 // blocks per SM the 4-slot ILU0 warp kernel is compiled for
#endif

namespace sfg {

namespace {

constexpr int kFBlock = 256;
constexpr int kMaxIluUpd = 8;  // ILU0: updates a lane holds in registers
constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ unsigned long long ftimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ double fsub_mul(double acc, double a, double b) {
  return __dsub_rn(acc, __dmul_rn(a, b));
}

__device__ __forceinline__ double resolve(unsigned long long w, const double* p, unsigned cap) {
  return is_sent_hi(w) ? poll_f64(p, cap) : __longlong_as_double((long long)w);
}

int grid_n(int64_t n) {
  int64_t b = (n + kFBlock - 1) / kFBlock;
  const int64_t cap = (int64_t)sm_count() * 16;
  return (int)std::max<int64_t>(1, std::min(b, cap));
}

// ---------------------------------------------------------------------------
// Inspector.  MODE 0 counts the updates of every factor position into cur[];
// MODE 1 appends them at cur[target]++ (cur = exclusive scan of the counts).
// One thread owns one task, i.e. every target position it writes, so the
// lists come out in the task's loop order without atomics.
// ---------------------------------------------------------------------------

// IC0 column k: for each L(k,j) (row view q ascending = j ascending), the
// rows of column j from k on that also occur in column k.
template <int MODE>
__global__ void k_ic0_updates(const int32_t* __restrict__ lc_ptr, const int32_t* __restrict__ lc_idx,
                              const int32_t* __restrict__ rv_ptr, const int32_t* __restrict__ rv_col,
                              const int32_t* __restrict__ rv_pos, int32_t n, int32_t* cur,
                              int32_t* __restrict__ oa, int32_t* __restrict__ ob) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int c0 = lc_ptr[k], c1 = lc_ptr[k + 1];
    for (int q = rv_ptr[k]; q < rv_ptr[k + 1]; ++q) {
      const int j = rv_col[q], pj = rv_pos[q], pe = lc_ptr[j + 1];
      int a = c0;
      for (int p = pj; p < pe && a < c1; ++p) {
        const int i = lc_idx[p];
        while (a < c1 && lc_idx[a] < i)
          ++a;
        if (a < c1 && lc_idx[a] == i) {
          if (MODE == 0) {
            ++cur[a];
          } else {
            const int e = cur[a]++;
            oa[e] = p;  // fac[p] = L(i,j)
            ob[e] = pj; // fac[pj] = L(k,j)
          }
        }
      }
    }
  }
}

// ILU0 row i: for each lower entry k (pivot step t, ascending), the upper
// entries U(k,j) of row k whose column j also occurs in row i after k.
template <int MODE>
__global__ void k_ilu0_updates(const int32_t* __restrict__ ar_ptr, const int32_t* __restrict__ ar_idx,
                               const int32_t* __restrict__ diag, int32_t n, int32_t* cur,
                               int32_t* __restrict__ oa, int32_t* __restrict__ ob) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int r0 = ar_ptr[i], r1 = ar_ptr[i + 1];
    for (int pa = r0; pa < r1; ++pa) {
      const int k = ar_idx[pa];
      if (k >= i)
        break;
      const int dk = diag[k];
      if (dk < 0) // missing pivot: reported by the executor
        continue;
      const int qe = ar_ptr[k + 1];
      int b = pa + 1;
      for (int q = dk + 1; q < qe && b < r1; ++q) {
        const int j = ar_idx[q];
        while (b < r1 && ar_idx[b] < j)
          ++b;
        if (b < r1 && ar_idx[b] == j) {
          if (MODE == 0) {
            ++cur[b];
          } else {
            const int e = cur[b]++;
            oa[e] = pa - r0; // pivot step
            ob[e] = q;       // fac[q] = U(k,j)
          }
        }
      }
    }
  }
}

__global__ void k_list_stats(const int32_t* __restrict__ tptr, int32_t n,
                             const int32_t* __restrict__ uptr, int64_t nnz, int32_t* out) {
  int mt = 0, mu = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    mt = max(mt, tptr[i + 1] - tptr[i]);
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nnz;
       p += (int64_t)gridDim.x * blockDim.x)
    mu = max(mu, uptr[p + 1] - uptr[p]);
  atomicMax(out, mt);
  atomicMax(out + 1, mu);
}

__global__ void k_sum64(const int32_t* __restrict__ v, int64_t n, unsigned long long* out) {
  unsigned long long acc = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    acc += (unsigned)v[i];
  for (int o = 16; o > 0; o >>= 1)
    acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0)
    atomicAdd(out, acc);
}

// Update lists are indexed with int32: a pattern whose total exceeds 2^31 - 1
// updates (they grow faster than nnz) gets no lists -- out.count = -1, and
// the *_warp_fits checks send the plan to the level-set executor.
template <typename CountK, typename FillK>
void build_lists(int32_t n, int64_t nnz, const int32_t* tptr, UpdateLists& out, cudaStream_t s,
                 CountK count, FillK fill) {
  DBuf<int32_t> cnt(nnz + 1);
  SFG_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int32_t) * (size_t)(nnz + 1), s));
  count(cnt.p);
  {
    DBuf<unsigned long long> tot(1);
    SFG_CUDA(cudaMemsetAsync(tot.p, 0, sizeof(unsigned long long), s));
    k_sum64<<<grid_n(nnz), kFBlock, 0, s>>>(cnt.p, nnz, tot.p);
    count_launch();
    unsigned long long h = 0;
    SFG_CUDA(cudaMemcpyAsync(&h, tot.p, sizeof(h), cudaMemcpyDeviceToHost, s));
    SFG_CUDA(cudaStreamSynchronize(s));
    if (h > (unsigned long long)INT32_MAX - 1) {
      out.count = -1;
      out.max_task = INT32_MAX;
      out.max_updates = INT32_MAX;
      return;
    }
  }
  out.ptr.alloc(nnz + 1);
  size_t bytes = 0;
  SFG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, cnt.p, out.ptr.p, nnz + 1, s));
  {
    DBuf<unsigned char> tmp((int64_t)bytes);
    SFG_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, cnt.p, out.ptr.p, nnz + 1, s));
  }
  int32_t total = 0;
  SFG_CUDA(cudaMemcpyAsync(&total, out.ptr.p + nnz, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  SFG_CUDA(cudaStreamSynchronize(s));
  out.count = total;
  out.a.alloc(total > 0 ? total : 1);
  out.b.alloc(total > 0 ? total : 1);
  SFG_CUDA(cudaMemcpyAsync(cnt.p, out.ptr.p, sizeof(int32_t) * (size_t)(nnz + 1),
                           cudaMemcpyDeviceToDevice, s));
  fill(cnt.p, out.a.p, out.b.p);
  DBuf<int32_t> st(2);
  SFG_CUDA(cudaMemsetAsync(st.p, 0, sizeof(int32_t) * 2, s));
  k_list_stats<<<grid_n(std::max<int64_t>(n, nnz)), kFBlock, 0, s>>>(tptr, n, out.ptr.p, nnz, st.p);
  count_launch();
  SFG_CUDA(cudaGetLastError());
  int32_t h[2];
  SFG_CUDA(cudaMemcpyAsync(h, st.p, sizeof(h), cudaMemcpyDeviceToHost, s));
  SFG_CUDA(cudaStreamSynchronize(s));
  out.max_task = h[0];
  out.max_updates = h[1];
}

// ---------------------------------------------------------------------------
// Executors.  One ticket = one task = one warp; lane a owns entry a of the
// column (IC0) or row (ILU0).  Tasks are claimed in the inspector's level
// order, so every producer a warp polls is already claimed (deadlock-free).
// ---------------------------------------------------------------------------

// IC0 column k (ic0_column, kernels.hpp:214-242), fused with the CSC-row
// solve x_k (trsv_csc_row, kernels.hpp:200-210) for combo 5 or with DSCAL
// applied on load (dscal_csc_col, kernels.hpp:281-286) for combo 7.
//   src 0: column k from lc_val; 1: scaled on load; 2: pre-scaled in work.
template <int COMBO>
__global__ void __launch_bounds__(kFBlock, COMBO == 5 ? SFG_IC5_MINB : SFG_IC7_MINB) k_ic0_warp(const ExecArgs A,
                                                      const int32_t* __restrict__ uptr,
                                                      const int32_t* __restrict__ usrc,
                                                      const int32_t* __restrict__ ulkj) {
  constexpr int CHU = COMBO == 5 ? SFG_IC5_CHU : SFG_IC7_CHU;
  const int lane = threadIdx.x & 31;
  const int64_t total = A.t_end - A.t_begin;
  const bool do_fac = COMBO == 5 ? (A.phase & 1) : (A.phase & 2);
  const bool do_solve = COMBO == 5 && (A.phase & 2);
  const int src = COMBO == 5 ? 0 : ((A.phase & 1) ? 1 : 2);
  const int fac_kernel = COMBO == 5 ? 1 : 2;
  const unsigned cap = A.sleep_cap;
  // next task claimed and its column header loaded during this one (see
  // k_ilu0_warp)
  unsigned long long nb = 0;
  if (lane == 0)
    nb = atomicAdd(A.counter, 1ull);
  long long c = (long long)__shfl_sync(FULL, nb, 0);
  int k_nx = 0, c0_nx = 0, c1_nx = 0, q0_nx = 0, q1_nx = 0;
  auto header = [&]() {
    k_nx = __ldg(A.order + A.t_begin + c);
    c0_nx = __ldg(A.lc_ptr + k_nx);
    c1_nx = __ldg(A.lc_ptr + k_nx + 1);
    if (do_solve) {
      q0_nx = __ldg(A.rv_ptr + k_nx);
      q1_nx = __ldg(A.rv_ptr + k_nx + 1);
    }
  };
  if (c < total)
    header();
  for (;;) {
    if (c >= total)
      break;
    const int k = k_nx;
    const int c0 = c0_nx;
    const int m = c1_nx - c0;
    const int q0 = q0_nx;
    const int q1 = q1_nx;
    unsigned long long* const ftr =
        SFG_FACT_TRACE && A.ftrace ? A.ftrace + (size_t)c * 5 : nullptr;
    if (ftr && lane == 0) {
      ftr[0] = (unsigned long long)k;
      ftr[1] = ftimer();
    }
    if (lane == 0)
      nb = atomicAdd(A.counter, 1ull);
    // the solve's first 32 operands L(k,j), x_j: loads in flight during the
    // factorization of column k
    unsigned long long wl = 0, wx = 0;
    int ql = -1, qx = -1;
    // the right-hand side of the solve row, in flight during the factorization too
    const double bk = do_solve ? __ldg(A.vin + k) : 0.0;
    if (do_solve && q0 + lane < q1) {
      ql = __ldg(A.rv_pos + q0 + lane);
      qx = __ldg(A.rv_col + q0 + lane);
      wl = ld_relaxed_u64(A.fac + ql);
      wx = ld_relaxed_u64(A.vout + qx);
    }
    double lkk;
    if (do_fac) {
      const int pa = c0 + lane;
      double acc = 0.0;
      int u0 = 0, u1 = 0;
      if (lane < m) {
        if (src == 0) {
          acc = __ldg(A.lc_val + pa);
        } else if (src == 1) {
          const int row = __ldg(A.lc_idx + pa);
          acc = __dmul_rn(__dmul_rn(__ldg(A.dvec + row), __ldg(A.lc_val + pa)), __ldg(A.dvec + k));
        } else {
          acc = __ldg(A.work + pa);
        }
        u0 = __ldg(uptr + pa);
        u1 = __ldg(uptr + pa + 1);
      }
#if SFG_IC_BUNROLL
      constexpr int kUnrollB = SFG_IC_BUNROLL;
#pragma unroll kUnrollB
#endif
      for (int u = u0; u < u1; u += CHU) {
        const int cnt = min(CHU, u1 - u);
        int ps[CHU], pl[CHU];
        unsigned long long ws[CHU], wk[CHU];
#pragma unroll
        for (int e = 0; e < CHU; ++e)
          if (e < cnt) {
            ps[e] = __ldg(usrc + u + e);
            pl[e] = __ldg(ulkj + u + e);
          }
#pragma unroll
        for (int e = 0; e < CHU; ++e)
          if (e < cnt) {
            ws[e] = ld_relaxed_u64(A.fac + ps[e]);
            wk[e] = ld_relaxed_u64(A.fac + pl[e]);
          }
        if constexpr (COMBO == 5) {
          // re-poll every still-unpublished word of the batch together (one
          // round trip per pass), so a word published while an earlier one
          // was awaited costs no extra trip: C2 0.53 -> 0.48 ms.  On C4's
          // long critical path (many warps waiting) the extra polling traffic
          // costs more than it saves (11.9 -> 13.4 ms), so COMBO 7 awaits
          // the updates one at a time (below).
          for (;;) {
            bool pending = false;
#pragma unroll
            for (int e = 0; e < CHU; ++e)
              pending |= e < cnt && (is_sent_hi(ws[e]) || is_sent_hi(wk[e]));
            if (!pending)
              break;
#pragma unroll
            for (int e = 0; e < CHU; ++e)
              if (e < cnt) {
                if (is_sent_hi(ws[e]))
                  ws[e] = ld_relaxed_u64(A.fac + ps[e]);
                if (is_sent_hi(wk[e]))
                  wk[e] = ld_relaxed_u64(A.fac + pl[e]);
              }
          }
#pragma unroll
          for (int e = 0; e < CHU; ++e)
            if (e < cnt)
              acc = fsub_mul(acc, __longlong_as_double((long long)wk[e]),
                             __longlong_as_double((long long)ws[e]));
        } else {
          // in order; an update whose words are still out spins on both of
          // them together, then the later stale words of the batch are
          // re-read once (their producers may have published meanwhile), so
          // words from the same producer cost one round trip, not one each
#pragma unroll
          for (int e = 0; e < CHU; ++e)
            if (e < cnt) {
              if (is_sent_hi(wk[e]) || is_sent_hi(ws[e])) {
                do {
                  if (is_sent_hi(wk[e]))
                    wk[e] = ld_relaxed_u64(A.fac + pl[e]);
                  if (is_sent_hi(ws[e]))
                    ws[e] = ld_relaxed_u64(A.fac + ps[e]);
                } while (is_sent_hi(wk[e]) || is_sent_hi(ws[e]));
#pragma unroll
                for (int f = e + 1; f < CHU; ++f)
                  if (f < cnt) {
                    if (is_sent_hi(wk[f]))
                      wk[f] = ld_relaxed_u64(A.fac + pl[f]);
                    if (is_sent_hi(ws[f]))
                      ws[f] = ld_relaxed_u64(A.fac + ps[f]);
                  }
              }
              acc = fsub_mul(acc, __longlong_as_double((long long)wk[e]),
                             __longlong_as_double((long long)ws[e]));
            }
        }
      }
      double l0 = 0.0;
      if (lane == 0) {
        if (acc <= 0.0)
          report_error(A.err, fac_kernel, k, k);
        l0 = __dsqrt_rn(acc);
      }
      lkk = __shfl_sync(FULL, l0, 0);
      if (ftr && lane == 0)
        ftr[2] = ftimer();
      // (a reciprocal formed after the square root and broadcast measured
      // slower than the lanes' own IEEE divisions: C4 15.5 vs 13.1 ms)
      if (lane < m)
        publish_f64(A.fac + pa, lane == 0 ? lkk : __ddiv_rn(acc, lkk));
      if (ftr) {
        __syncwarp();
        if (lane == 0)
          ftr[3] = ftimer();
      }
    } else {
      lkk = do_solve ? poll_f64(A.fac + c0, cap) : 0.0;
    }
    if (do_solve) {
      double acc2 = bk;
      for (int qb = q0; qb < q1; qb += 32) {
        double lv = 0.0, xv = 0.0;
        if (qb + lane < q1) {
          if (qb != q0) {
            ql = __ldg(A.rv_pos + qb + lane);
            qx = __ldg(A.rv_col + qb + lane);
            wl = ld_relaxed_u64(A.fac + ql);
            wx = ld_relaxed_u64(A.vout + qx);
          }
          // L(k,j) and x_j come from the same task j: await them together
          while (is_sent_hi(wl) || is_sent_hi(wx)) {
            if (is_sent_hi(wl))
              wl = ld_relaxed_u64(A.fac + ql);
            if (is_sent_hi(wx))
              wx = ld_relaxed_u64(A.vout + qx);
          }
          lv = __longlong_as_double((long long)wl);
          xv = __longlong_as_double((long long)wx);
        }
        const int cnt = min(32, q1 - qb);
        // each lane rounds its own product; the serial chain only shuffles
        // and subtracts (the same separately rounded product and difference
        // as fsub_mul, so the order and result are the reference's)
        const double pr = __dmul_rn(lv, xv);
#if SFG_IC_UNROLL
        constexpr int kUnrollS = SFG_IC_UNROLL;
#pragma unroll kUnrollS
#endif
        for (int t = 0; t < cnt; ++t)
          acc2 = __dsub_rn(acc2, __shfl_sync(FULL, pr, t));
      }
      if (lane == 0) {
        if (lkk == 0.0)
          report_error(A.err, 2, k, k);
        publish_f64(A.vout + k, __ddiv_rn(acc2, lkk));
        if (ftr)
          ftr[4] = ftimer();
      }
    }
    // (prefetching the next header across this task's phases, as k_ilu0_warp
    // does, measured slower here: C2 +3 %, C4 +1 %; fetching the ticket
    // before the square root +50 % on C4)
    c = (long long)__shfl_sync(FULL, nb, 0);
    if (c < total)
      header();
  }
}

// Per-ticket task record of the IC0 executors, in claim order: {column k,
// lc_ptr[k], lc_ptr[k+1], rv_ptr[k]}, {rv_ptr[k+1], -, -, -}.  One load by
// ticket number replaces the order -> pointer chain at the start of a task.
__global__ void k_ic0_task_records(const int32_t* __restrict__ order,
                                   const int32_t* __restrict__ lc_ptr,
                                   const int32_t* __restrict__ rv_ptr, int64_t ntask,
                                   int4* __restrict__ rec) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < ntask;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int k = order[t];
    rec[2 * t] = make_int4(k, lc_ptr[k], lc_ptr[k + 1], rv_ptr[k]);
    rec[2 * t + 1] = make_int4(rv_ptr[k + 1], 0, 0, 0);
  }
}

// Fused IC0 -> solve (combo 5, both kernels in one launch) with the operands
// of the NEXT task loaded during the current one.  A warp holds three
// tickets in claim order: the task it runs, the next one (its record loaded
// a task ago, its per-lane operands -- column values, update-list bounds, the
// solve row's entries, the right-hand side -- loaded between this task's
// factorization and its solve) and a third whose record is in flight.  A
// task then starts with its update-list and factor-word loads instead of
// five dependent round trips.  Tickets are claimed in increasing order and
// run in that order, so the smallest unfinished ticket is always running:
// deadlock-free like k_ic0_warp.  Arithmetic and error reporting are
// k_ic0_warp<5>'s.
struct IcLane {
  double acc, bk;
  int u0, u1, ql, qx;
};

template <int CHU>
__global__ void __launch_bounds__(kFBlock, 3) k_ic0_pipe(const ExecArgs A,
                                                         const int32_t* __restrict__ uptr,
                                                         const int32_t* __restrict__ usrc,
                                                         const int32_t* __restrict__ ulkj,
                                                         const int4* __restrict__ trec) {
  const int lane = threadIdx.x & 31;
  const int64_t total = A.t_end - A.t_begin;
  auto claim = [&]() {
    unsigned long long nb = 0;
    if (lane == 0)
      nb = atomicAdd(A.counter, 1ull);
    return (long long)__shfl_sync(FULL, nb, 0);
  };
  auto load_rec = [&](long long t, int4& a, int4& b) {
    if (t < total) {
      a = __ldg(trec + 2 * (A.t_begin + t));
      b = __ldg(trec + 2 * (A.t_begin + t) + 1);
    }
  };
  auto load_lane = [&](const int4& a, const int4& b, IcLane& L) {
    const int c0 = a.y, m = a.z - a.y, q0 = a.w, q1 = b.x;
    L.acc = 0.0;
    L.u0 = L.u1 = 0;
    L.ql = L.qx = -1;
    if (lane < m) {
      L.acc = __ldg(A.lc_val + c0 + lane);
      L.u0 = __ldg(uptr + c0 + lane);
      L.u1 = __ldg(uptr + c0 + lane + 1);
    }
    if (q0 + lane < q1) {
      L.ql = __ldg(A.rv_pos + q0 + lane);
      L.qx = __ldg(A.rv_col + q0 + lane);
    }
    L.bk = __ldg(A.vin + a.x);
  };
  long long t0 = claim(), t1 = claim();
  int4 ha0 = make_int4(0, 0, 0, 0), hb0 = ha0, ha1 = ha0, hb1 = ha0;
  load_rec(t0, ha0, hb0);
  load_rec(t1, ha1, hb1);
  IcLane L0{0.0, 0.0, 0, 0, -1, -1}, L1 = L0;
  if (t0 < total)
    load_lane(ha0, hb0, L0);
  while (t0 < total) {
    unsigned long long nb = 0;
    if (lane == 0)
      nb = atomicAdd(A.counter, 1ull);
    const int k = ha0.x, c0 = ha0.y, m = ha0.z - ha0.y, q0 = ha0.w, q1 = hb0.x;
    // the solve's first 32 operands L(k,j), x_j: in flight during the factorization
    int ql = L0.ql, qx = L0.qx;
    unsigned long long wl = 0, wx = 0;
    if (ql >= 0) {
      wl = ld_relaxed_u64(A.fac + ql);
      wx = ld_relaxed_u64(A.vout + qx);
    }
    const int pa = c0 + lane;
    double acc = L0.acc;
    const int u0 = L0.u0, u1 = L0.u1;
    for (int u = u0; u < u1; u += CHU) {
      const int cnt = min(CHU, u1 - u);
      int ps[CHU], pl[CHU];
      unsigned long long ws[CHU], wk[CHU];
#pragma unroll
      for (int e = 0; e < CHU; ++e)
        if (e < cnt) {
          ps[e] = __ldg(usrc + u + e);
          pl[e] = __ldg(ulkj + u + e);
        }
#pragma unroll
      for (int e = 0; e < CHU; ++e)
        if (e < cnt) {
          ws[e] = ld_relaxed_u64(A.fac + ps[e]);
          wk[e] = ld_relaxed_u64(A.fac + pl[e]);
        }
      for (;;) {
        bool pending = false;
#pragma unroll
        for (int e = 0; e < CHU; ++e)
          pending |= e < cnt && (is_sent_hi(ws[e]) || is_sent_hi(wk[e]));
        if (!pending)
          break;
#pragma unroll
        for (int e = 0; e < CHU; ++e)
          if (e < cnt) {
            if (is_sent_hi(ws[e]))
              ws[e] = ld_relaxed_u64(A.fac + ps[e]);
            if (is_sent_hi(wk[e]))
              wk[e] = ld_relaxed_u64(A.fac + pl[e]);
          }
      }
#pragma unroll
      for (int e = 0; e < CHU; ++e)
        if (e < cnt)
          acc = fsub_mul(acc, __longlong_as_double((long long)wk[e]),
                         __longlong_as_double((long long)ws[e]));
    }
    double l0 = 0.0;
    if (lane == 0) {
      if (acc <= 0.0)
        report_error(A.err, 1, k, k);
      l0 = __dsqrt_rn(acc);
    }
    const double lkk = __shfl_sync(FULL, l0, 0);
    if (lane < m)
      publish_f64(A.fac + pa, lane == 0 ? lkk : __ddiv_rn(acc, lkk));
    // the next task's per-lane operands (its record arrived a task ago)
    if (t1 < total)
      load_lane(ha1, hb1, L1);
    // solve row k (trsv_csc_row, kernels.hpp:200-210)
    double acc2 = L0.bk;
    for (int qb = q0; qb < q1; qb += 32) {
      double lv = 0.0, xv = 0.0;
      if (qb + lane < q1) {
        if (qb != q0) {
          ql = __ldg(A.rv_pos + qb + lane);
          qx = __ldg(A.rv_col + qb + lane);
          wl = ld_relaxed_u64(A.fac + ql);
          wx = ld_relaxed_u64(A.vout + qx);
        }
        // L(k,j) and x_j come from the same task j: await them together
        while (is_sent_hi(wl) || is_sent_hi(wx)) {
          if (is_sent_hi(wl))
            wl = ld_relaxed_u64(A.fac + ql);
          if (is_sent_hi(wx))
            wx = ld_relaxed_u64(A.vout + qx);
        }
        lv = __longlong_as_double((long long)wl);
        xv = __longlong_as_double((long long)wx);
      }
      const int cnt = min(32, q1 - qb);
      const double pr = __dmul_rn(lv, xv);
#if SFG_IC_UNROLL
      constexpr int kUnrollS = SFG_IC_UNROLL;
#pragma unroll kUnrollS
#endif
      for (int t = 0; t < cnt; ++t)
        acc2 = __dsub_rn(acc2, __shfl_sync(FULL, pr, t));
    }
    if (lane == 0) {
      if (lkk == 0.0)
        report_error(A.err, 2, k, k);
      publish_f64(A.vout + k, __ddiv_rn(acc2, lkk));
    }
    // rotate the ticket queue
    t0 = t1;
    ha0 = ha1;
    hb0 = hb1;
    L0 = L1;
    t1 = (long long)__shfl_sync(FULL, nb, 0);
    load_rec(t1, ha1, hb1);
  }
}

// IKJ ILU0 row i (ilu0_row, kernels.hpp:246-272) fused with the unit-lower
// solve y_i (trsv_csr_unit_row, kernels.hpp:184-196).  Pivot step t is the
// t-th lower entry k_t of row i: lane t forms l_{i,k_t} = a_{i,k_t} / u_{k_t k_t}
// once the updates of steps < t have reached it, the multiplier is broadcast,
// and every lane holding a matching U(k_t, j) applies it.  The reciprocals of
// all pivots are formed before the first step, off the serial chain.
// COMBO 3 (DSCAL -> ILU0): no solve; the row is scaled on load,
// (d_i * a_ij) * d_j (dscal_csr_row, kernels.hpp:274-279), when fused, or
// read from `work` after a separate DSCAL launch.
// MAXU: update slots a lane holds in registers (the pattern's maximum, 4 or
// 8); the 4-slot build is compiled for 3 resident blocks per SM (80
// registers, no spills): C3 1.545 -> 1.436 ms
template <int COMBO, int MAXU>
__global__ void __launch_bounds__(kFBlock, MAXU <= 4 ? SFG_ILU_MINB4 : 1) k_ilu0_warp(const ExecArgs A,
                                                       const int32_t* __restrict__ uptr,
                                                       const int32_t* __restrict__ ustep,
                                                       const int32_t* __restrict__ usrc) {
  const int lane = threadIdx.x & 31;
  const int64_t total = A.t_end - A.t_begin;
  const bool do_fac = COMBO == 6 ? (A.phase & 1) : (A.phase & 2);
  const bool do_solve = COMBO == 6 && (A.phase & 2);
  const int src = COMBO == 6 ? 0 : ((A.phase & 1) ? 1 : 2);
  const int fac_kernel = COMBO == 6 ? 1 : 2;
  const unsigned cap = A.sleep_cap;
  // The next task is claimed while this one runs and its row header is
  // loaded then, so a task starts with its per-lane loads instead of three
  // dependent round trips (claim, order, row pointers).  Progress holds: the
  // lowest unfinished ticket is always some warp's current task.
  unsigned long long nb = 0;
  if (lane == 0)
    nb = atomicAdd(A.counter, 1ull);
  long long c = (long long)__shfl_sync(FULL, nb, 0);
  int i_nx = 0, r0_nx = 0, r1_nx = 0;
  if (c < total) {
    i_nx = __ldg(A.order + A.t_begin + c);
    r0_nx = __ldg(A.ar_ptr + i_nx);
    r1_nx = __ldg(A.ar_ptr + i_nx + 1);
  }
  for (;;) {
    if (c >= total)
      break;
    const int i = i_nx;
    const int r0 = r0_nx;
    const int m = r1_nx - r0;
    unsigned long long* const ftr =
        SFG_FACT_TRACE && A.ftrace ? A.ftrace + (size_t)c * 5 : nullptr;
    if (ftr && lane == 0) {
      ftr[0] = (unsigned long long)i;
      ftr[1] = ftimer();
    }
    if (lane == 0)
      nb = atomicAdd(A.counter, 1ull);
    long long c_next = -1;
    const int pb = r0 + lane;
    const int col = lane < m ? __ldg(A.ar_idx + pb) : 0x7fffffff;
    const bool lower = col < i;
    const int nl = __popc(__ballot_sync(FULL, lower)); // lower lanes are 0 .. nl-1
    unsigned long long wx = 0;
    if (do_solve && lower)
      wx = ld_relaxed_u64(A.vout + col);
    double acc2 = do_solve ? __ldg(A.vin + i) : 0.0;
    if (do_fac) {
      double acc = 0.0;
      if (lane < m)
        acc = src == 0   ? __ldg(A.ar_val + pb)
              : src == 1 ? __dmul_rn(__dmul_rn(__ldg(A.dvec + i), __ldg(A.ar_val + pb)),
                                     __ldg(A.dvec + col))
                         : __ldg(A.work + pb);
      const int dk = lower ? __ldg(A.diag + col) : -1;
      unsigned long long wp = 0;
      if (dk >= 0)
        wp = ld_relaxed_u64(A.fac + dk);
      int nu = 0, ub = 0;
      if (lane < m) {
        ub = __ldg(uptr + pb);
        nu = __ldg(uptr + pb + 1) - ub;
      }
      int st[MAXU];
      int sq[MAXU];
      unsigned long long wu[MAXU];
#pragma unroll
      for (int e = 0; e < MAXU; ++e) {
        st[e] = -1;
        if (e < nu) {
          st[e] = __ldg(ustep + ub + e);
          sq[e] = __ldg(usrc + ub + e);
        }
      }
#pragma unroll
      for (int e = 0; e < MAXU; ++e)
        if (e < nu)
          wu[e] = ld_relaxed_u64(A.fac + sq[e]);
      // all of this lane's words re-polled together until published; the
      // solve's x_col (published by the same task as U(col, .)) with them
      const bool want_x = do_solve && lower;
      for (;;) {
        bool pending = (dk >= 0 && is_sent_hi(wp)) || (want_x && is_sent_hi(wx));
#pragma unroll
        for (int e = 0; e < MAXU; ++e)
          pending |= e < nu && is_sent_hi(wu[e]);
        if (!pending)
          break;
        if (dk >= 0 && is_sent_hi(wp))
          wp = ld_relaxed_u64(A.fac + dk);
        if (want_x && is_sent_hi(wx))
          wx = ld_relaxed_u64(A.vout + col);
#pragma unroll
        for (int e = 0; e < MAXU; ++e)
          if (e < nu && is_sent_hi(wu[e]))
            wu[e] = ld_relaxed_u64(A.fac + sq[e]);
      }
      // the next task's header, one dependent load per phase of this task
      // (ticket after the poll loop, row pointers after the pivot steps), so
      // it is in registers when this task ends
      c_next = (long long)__shfl_sync(FULL, nb, 0);
      if (c_next < total)
        i_nx = __ldg(A.order + A.t_begin + c_next);
      double uv[MAXU];
#pragma unroll
      for (int e = 0; e < MAXU; ++e)
        uv[e] = e < nu ? __longlong_as_double((long long)wu[e]) : 0.0;
      if (ftr) {
        __syncwarp();
        if (lane == 0)
          ftr[2] = ftimer();
      }
      const double piv = dk >= 0 ? __longlong_as_double((long long)wp) : 0.0;
      const double rcp = __drcp_rn(piv);
      const double xk = want_x ? __longlong_as_double((long long)wx) : 0.0;
#if SFG_ILU_UNROLL
      constexpr int kUnroll = SFG_ILU_UNROLL;
#pragma unroll kUnroll
#endif
      for (int t = 0; t < nl; ++t) {
        if (lane == t) {
          if (dk < 0 || piv == 0.0)
            report_error(A.err, fac_kernel, i, col);
          acc = div_with_rcp(acc, piv, rcp);
        }
        const double lik = __shfl_sync(FULL, acc, t);
#pragma unroll
        for (int e = 0; e < MAXU; ++e)
          if (st[e] == t)
            acc = fsub_mul(acc, lik, uv[e]);
        if (do_solve)
          acc2 = fsub_mul(acc2, lik, __shfl_sync(FULL, xk, t));
      }
      if (c_next < total) {
        r0_nx = __ldg(A.ar_ptr + i_nx);
        r1_nx = __ldg(A.ar_ptr + i_nx + 1);
      }
      if (lane < m)
        publish_f64(A.fac + pb, acc);
      if (ftr) {
        __syncwarp();
        if (lane == 0)
          ftr[3] = ftimer();
      }
    } else if (do_solve) { // unit solve alone (unfused second launch)
      double lv = 0.0, xk = 0.0;
      if (lower) {
        lv = poll_f64(A.fac + pb, cap);
        xk = resolve(wx, A.vout + col, cap);
      }
      const double pr = __dmul_rn(lv, xk); // per-lane product, as in k_ic0_warp
#if SFG_IC_UNROLL
      constexpr int kUnrollU = SFG_IC_UNROLL;
#pragma unroll kUnrollU
#endif
      for (int t = 0; t < nl; ++t)
        acc2 = __dsub_rn(acc2, __shfl_sync(FULL, pr, t));
    }
    if (do_solve && lane == 0) {
      publish_f64(A.vout + i, acc2);
      if (ftr)
        ftr[4] = ftimer();
    }
    if (c_next < 0) { // header not prefetched (solve-only launch)
      c_next = (long long)__shfl_sync(FULL, nb, 0);
      if (c_next < total) {
        i_nx = __ldg(A.order + A.t_begin + c_next);
        r0_nx = __ldg(A.ar_ptr + i_nx);
        r1_nx = __ldg(A.ar_ptr + i_nx + 1);
      }
    }
    c = c_next;
  }
}

// ILU0 rows packed PK = 32/SEG to a warp (SEG lanes per row, every row of a
// pack from the same dependency level, so no row waits on a packmate).  The
// same lane roles as k_ilu0_warp inside each segment; the waits are one
// warp-uniform loop -- every segment re-polls its own pending words in the
// same pass -- and the pivot steps run to the widest row's lower count, so
// a warp issues each instruction once for PK rows.
template <int COMBO, int MAXU, int SEG>
__global__ void __launch_bounds__(kFBlock, SFG_ILU_MINB4) k_ilu0_pack(const ExecArgs A,
                                                         const int32_t* __restrict__ uptr,
                                                         const int32_t* __restrict__ ustep,
                                                         const int32_t* __restrict__ usrc,
                                                         const int32_t* __restrict__ pack_ptr,
                                                         int32_t npack) {
  constexpr int PK = 32 / SEG;
  const int lane = threadIdx.x & 31;
  const int seg = lane / SEG;
  const int sl = lane % SEG;
  const unsigned smask = (SEG == 32 ? FULL : ((1u << SEG) - 1u)) << (seg * SEG);
  const bool do_fac = COMBO == 6 ? (A.phase & 1) : (A.phase & 2);
  const bool do_solve = COMBO == 6 && (A.phase & 2);
  const int src = COMBO == 6 ? 0 : ((A.phase & 1) ? 1 : 2);
  const int fac_kernel = COMBO == 6 ? 1 : 2;
  for (;;) {
    unsigned long long w0 = 0;
    if (lane == 0)
      w0 = atomicAdd(A.counter, 1ull);
    const long long pk = (long long)__shfl_sync(FULL, w0, 0);
    if (pk >= npack)
      break;
    const int t0 = __ldg(pack_ptr + pk), t1 = __ldg(pack_ptr + pk + 1);
    const int tk = t0 + seg;
    const bool task = tk < t1;
    int i = 0, r0 = 0, m = 0;
    if (task) {
      i = __ldg(A.order + A.t_begin + tk);
      r0 = __ldg(A.ar_ptr + i);
      m = __ldg(A.ar_ptr + i + 1) - r0;
    }
    const int pb = r0 + sl;
    const bool mine = task && sl < m;
    const int col = mine ? __ldg(A.ar_idx + pb) : 0x7fffffff;
    const bool lower = col < i;
    const int nl = __popc(__ballot_sync(FULL, lower) & smask); // lower lanes: sl 0 .. nl-1
    const int nlmax = __reduce_max_sync(FULL, nl);
    unsigned long long wx = 0;
    const bool want_x = do_solve && lower;
    if (want_x)
      wx = ld_relaxed_u64(A.vout + col);
    double acc2 = (do_solve && task) ? __ldg(A.vin + i) : 0.0;
    if (do_fac) {
      double acc = 0.0;
      if (mine)
        acc = src == 0   ? __ldg(A.ar_val + pb)
              : src == 1 ? __dmul_rn(__dmul_rn(__ldg(A.dvec + i), __ldg(A.ar_val + pb)),
                                     __ldg(A.dvec + col))
                         : __ldg(A.work + pb);
      const int dk = lower ? __ldg(A.diag + col) : -1;
      unsigned long long wp = 0;
      if (dk >= 0)
        wp = ld_relaxed_u64(A.fac + dk);
      int nu = 0, ub = 0;
      if (mine) {
        ub = __ldg(uptr + pb);
        nu = __ldg(uptr + pb + 1) - ub;
      }
      int st[MAXU];
      int sq[MAXU];
      unsigned long long wu[MAXU];
#pragma unroll
      for (int e = 0; e < MAXU; ++e) {
        st[e] = -1;
        if (e < nu) {
          st[e] = __ldg(ustep + ub + e);
          sq[e] = __ldg(usrc + ub + e);
        }
      }
#pragma unroll
      for (int e = 0; e < MAXU; ++e)
        if (e < nu)
          wu[e] = ld_relaxed_u64(A.fac + sq[e]);
      // one warp-uniform wait: every lane re-reads its own pending words in
      // the same pass until no lane of the warp has any
      for (;;) {
        bool pending = (dk >= 0 && is_sent_hi(wp)) || (want_x && is_sent_hi(wx));
#pragma unroll
        for (int e = 0; e < MAXU; ++e)
          pending |= e < nu && is_sent_hi(wu[e]);
        if (!__any_sync(FULL, pending))
          break;
        if (dk >= 0 && is_sent_hi(wp))
          wp = ld_relaxed_u64(A.fac + dk);
        if (want_x && is_sent_hi(wx))
          wx = ld_relaxed_u64(A.vout + col);
#pragma unroll
        for (int e = 0; e < MAXU; ++e)
          if (e < nu && is_sent_hi(wu[e]))
            wu[e] = ld_relaxed_u64(A.fac + sq[e]);
      }
      double uv[MAXU];
#pragma unroll
      for (int e = 0; e < MAXU; ++e)
        uv[e] = e < nu ? __longlong_as_double((long long)wu[e]) : 0.0;
      const double piv = dk >= 0 ? __longlong_as_double((long long)wp) : 0.0;
      const double rcp = __drcp_rn(piv);
      const double xk = want_x ? __longlong_as_double((long long)wx) : 0.0;
      const int base = seg * SEG;
#pragma unroll 2
      for (int t = 0; t < nlmax; ++t) {
        if (sl == t && t < nl) {
          if (dk < 0 || piv == 0.0)
            report_error(A.err, fac_kernel, i, col);
          acc = div_with_rcp(acc, piv, rcp);
        }
        const double lik = __shfl_sync(FULL, acc, base + t);
        if (t < nl) {
#pragma unroll
          for (int e = 0; e < MAXU; ++e)
            if (st[e] == t)
              acc = fsub_mul(acc, lik, uv[e]);
          if (do_solve)
            acc2 = fsub_mul(acc2, lik, __shfl_sync(FULL, xk, base + t));
        } else if (do_solve) {
          (void)__shfl_sync(FULL, xk, base + t);
        }
      }
      if (mine)
        publish_f64(A.fac + pb, acc);
    } else if (do_solve) { // unit solve alone (unfused second launch)
      double lv = 0.0, xk = 0.0;
      if (lower) {
        lv = poll_f64(A.fac + pb, 0);
        xk = resolve(wx, A.vout + col, 0);
      }
      const double pr = __dmul_rn(lv, xk);
      const int base = seg * SEG;
      for (int t = 0; t < nlmax; ++t) {
        const double v = __shfl_sync(FULL, pr, base + t);
        if (t < nl)
          acc2 = __dsub_rn(acc2, v);
      }
    }
    if (do_solve && task && sl == 0)
      publish_f64(A.vout + i, acc2);
  }
}

template <typename K> void launch_warp_tasks(K kernel, const ExecArgs& a, const UpdateLists& up,
                                             cudaStream_t s) {
  const int64_t total = a.t_end - a.t_begin;
  if (total <= 0)
    return;
  int per_sm = 0;
  SFG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kFBlock, 0));
  per_sm = std::max(per_sm, 1);
  if (a.blocks_per_sm > 0 && a.blocks_per_sm < per_sm)
    per_sm = a.blocks_per_sm;
  int64_t blocks = (total + (kFBlock / 32) - 1) / (kFBlock / 32);
  blocks = std::min<int64_t>(blocks, (int64_t)per_sm * sm_count());
  kernel<<<(unsigned)blocks, kFBlock, 0, s>>>(a, up.ptr.p, up.a.p, up.b.p);
  count_launch();
  SFG_CUDA(cudaGetLastError());
}

} // namespace

void build_ic0_updates(const int32_t* lc_ptr, const int32_t* lc_idx, const int32_t* rv_ptr,
                       const int32_t* rv_col, const int32_t* rv_pos, int32_t n, int64_t nnz,
                       UpdateLists& out, cudaStream_t s) {
  const int g = grid_n(n);
  build_lists(
      n, nnz, lc_ptr, out, s,
      [&](int32_t* cnt) {
        k_ic0_updates<0><<<g, kFBlock, 0, s>>>(lc_ptr, lc_idx, rv_ptr, rv_col, rv_pos, n, cnt,
                                               nullptr, nullptr);
        count_launch();
        SFG_CUDA(cudaGetLastError());
      },
      [&](int32_t* cur, int32_t* oa, int32_t* ob) {
        k_ic0_updates<1><<<g, kFBlock, 0, s>>>(lc_ptr, lc_idx, rv_ptr, rv_col, rv_pos, n, cur, oa, ob);
        count_launch();
        SFG_CUDA(cudaGetLastError());
      });
}

void build_ilu0_updates(const int32_t* ar_ptr, const int32_t* ar_idx, const int32_t* diag,
                        int32_t n, int64_t nnz, UpdateLists& out, cudaStream_t s) {
  const int g = grid_n(n);
  build_lists(
      n, nnz, ar_ptr, out, s,
      [&](int32_t* cnt) {
        k_ilu0_updates<0><<<g, kFBlock, 0, s>>>(ar_ptr, ar_idx, diag, n, cnt, nullptr, nullptr);
        count_launch();
        SFG_CUDA(cudaGetLastError());
      },
      [&](int32_t* cur, int32_t* oa, int32_t* ob) {
        k_ilu0_updates<1><<<g, kFBlock, 0, s>>>(ar_ptr, ar_idx, diag, n, cur, oa, ob);
        count_launch();
        SFG_CUDA(cudaGetLastError());
      });
}

int fact_warps_per_block() { return kFBlock / 32; }

void build_packs(const std::vector<int64_t>& wave_ptr, int32_t seg, UpdateLists& up) {
  up.seg = seg;
  const int32_t pk = 32 / seg;
  std::vector<int32_t> pp;
  for (size_t w = 0; w + 1 < wave_ptr.size(); ++w)
    for (int64_t a = wave_ptr[w]; a < wave_ptr[w + 1]; a += pk)
      pp.push_back((int32_t)a);
  pp.push_back(wave_ptr.empty() ? 0 : (int32_t)wave_ptr.back());
  up.npack = (int32_t)pp.size() - 1;
  up.pack_ptr.alloc((int64_t)pp.size());
  SFG_CUDA(cudaMemcpy(up.pack_ptr.p, pp.data(), sizeof(int32_t) * pp.size(), cudaMemcpyHostToDevice));
}

bool ic0_warp_fits(const UpdateLists& up) { return up.count >= 0 && up.max_task <= 32; }
bool ilu0_warp_fits(const UpdateLists& up) {
  return up.count >= 0 && up.max_task <= 32 && up.max_updates <= kMaxIluUpd;
}

template <typename K> void launch_pack_tasks(K kernel, const ExecArgs& a, const UpdateLists& up,
                                             cudaStream_t s) {
  if (up.npack <= 0)
    return;
  int per_sm = 0;
  SFG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kFBlock, 0));
  per_sm = std::max(per_sm, 1);
  if (a.blocks_per_sm > 0 && a.blocks_per_sm < per_sm)
    per_sm = a.blocks_per_sm;
  int64_t blocks = ((int64_t)up.npack + (kFBlock / 32) - 1) / (kFBlock / 32);
  blocks = std::min<int64_t>(blocks, (int64_t)per_sm * sm_count());
  kernel<<<(unsigned)blocks, kFBlock, 0, s>>>(a, up.ptr.p, up.a.p, up.b.p, up.pack_ptr.p, up.npack);
  count_launch();
  SFG_CUDA(cudaGetLastError());
}

void launch_ic0_warp(int combo, const ExecArgs& a, const UpdateLists& up, cudaStream_t s) {
  static const bool pipe_off = getenv("SFG_IC5_PIPE") && atoi(getenv("SFG_IC5_PIPE")) == 0;
  if (combo == 5 && a.phase == 3 && !a.ftrace && !pipe_off && a.t_begin == 0) {
    // the fused launch: task records in claim order, operands one task ahead
    const int64_t total = a.t_end - a.t_begin;
    if (total <= 0)
      return;
    if (up.trec.n < 8 * total) {
      up.trec.alloc(8 * total);
      k_ic0_task_records<<<grid_n(total), kFBlock, 0, s>>>(a.order, a.lc_ptr, a.rv_ptr, total,
                                                          reinterpret_cast<int4*>(up.trec.p));
      count_launch();
      SFG_CUDA(cudaGetLastError());
    }
    auto kernel = k_ic0_pipe<SFG_IC5_CHU>;
    int per_sm = 0;
    SFG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kFBlock, 0));
    per_sm = std::max(per_sm, 1);
    if (a.blocks_per_sm > 0 && a.blocks_per_sm < per_sm)
      per_sm = a.blocks_per_sm;
    int64_t blocks = (total + (kFBlock / 32) - 1) / (kFBlock / 32);
    blocks = std::min<int64_t>(blocks, (int64_t)per_sm * sm_count());
    kernel<<<(unsigned)blocks, kFBlock, 0, s>>>(a, up.ptr.p, up.a.p, up.b.p,
                                                reinterpret_cast<const int4*>(up.trec.p));
    count_launch();
    SFG_CUDA(cudaGetLastError());
    return;
  }
  if (combo == 5)
    launch_warp_tasks(k_ic0_warp<5>, a, up, s);
  else
    launch_warp_tasks(k_ic0_warp<7>, a, up, s);
}

void launch_ilu0_warp(int combo, const ExecArgs& a, const UpdateLists& up, cudaStream_t s) {
  if (up.seg == 8 && up.max_updates <= 4) {
    if (combo == 3)
      launch_pack_tasks(k_ilu0_pack<3, 4, 8>, a, up, s);
    else
      launch_pack_tasks(k_ilu0_pack<6, 4, 8>, a, up, s);
    return;
  }
  if (up.seg == 16 && up.max_updates <= 4) {
    if (combo == 3)
      launch_pack_tasks(k_ilu0_pack<3, 4, 16>, a, up, s);
    else
      launch_pack_tasks(k_ilu0_pack<6, 4, 16>, a, up, s);
    return;
  }
  const bool small = up.max_updates <= 4 && !getenv("SFG_ILU_MAXU8");
  if (combo == 3)
    small ? launch_warp_tasks(k_ilu0_warp<3, 4>, a, up, s) : launch_warp_tasks(k_ilu0_warp<3, 8>, a, up, s);
  else
    small ? launch_warp_tasks(k_ilu0_warp<6, 4>, a, up, s) : launch_warp_tasks(k_ilu0_warp<6, 8>, a, up, s);
}

} // namespace sfg
