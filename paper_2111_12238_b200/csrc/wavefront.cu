// wavefront.cu -- the joint-DAG wavefront executor (execute_joint_wavefront,
// executor.hpp:465-507; level sets from build_wavefront_schedule,
// executor.hpp:209-229).
//
// The paper's level-set baseline: every level of the joint DAG of the pair is
// one s-partition, the levels run one after another with a barrier between
// them, and the entries of a level -- kernel-1 and kernel-2 iterations mixed,
// ascending vertex id -- are spread over all threads.  On the GPU this is one
// persistent cooperative launch: a thread per (entry, system) runs the
// reference's iteration body sequentially, then the whole grid meets at a
// software grid barrier.  Every read of a value produced in the launch goes
// through L2 (ld.global.cg), so the barrier's release/acquire makes it
// visible; the bodies need no polling.
//
// Arithmetic is the reference's (kernels.hpp:145-286): storage-order
// accumulation with separately rounded products, IEEE division and square
// root.  The one exception is combo 4's CSC SpMV scatter, which the reference
// itself accumulates with atomic adds in any order (kernels.hpp:160-168,
// tolerance 1e-13 in test_kernels.cpp:395-396).
#include <cooperative_groups.h>

#include "common.cuh"
#include "executor.cuh"
#include "internal.hpp"

#include <algorithm>

namespace sfg {

namespace {

constexpr int kBlock = 256;

struct WaveArgs {
  ExecArgs a;
  int combo = 0;
  const int32_t* verts = nullptr; // joint vertices in level order
  const int64_t* lptr = nullptr;  // level boundaries (nlev + 1)
  int32_t nlev = 0;
  const int32_t* m_ptr = nullptr; // A in CSC (combo 4's spmv_csc_col)
  const int32_t* m_idx = nullptr;
  const double* m_val = nullptr;
};

__device__ __forceinline__ double ld_cg(const double* p) { return __ldcg(p); }
__device__ __forceinline__ double fsub_mul(double acc, double a, double b) {
  return __dsub_rn(acc, __dmul_rn(a, b));
}

// trsv_csr_row (kernels.hpp:171-181) over CSR rows with the diagonal last
__device__ void trsv_row(int r, int s, int S, const int32_t* ptr, const int32_t* idx,
                         const double* val, double rhs, double* x, unsigned long long* err,
                         int kernel, int seqpos) {
  const int e = __ldg(ptr + r + 1) - 1;
  double acc = rhs;
  for (int p = __ldg(ptr + r); p < e; ++p)
    acc = fsub_mul(acc, __ldg(val + (size_t)p * S + s), ld_cg(x + (size_t)__ldg(idx + p) * S + s));
  const double d = __ldg(val + (size_t)e * S + s);
  if (d == 0.0)
    report_error(err, kernel, seqpos, r);
  x[(size_t)r * S + s] = __ddiv_rn(acc, d);
}

// ic0_column (kernels.hpp:214-242): the dense marker becomes a merge of
// column k's sorted rows with column j's rows from L(k,j) on.  The column's
// initial values come from lc_val (combo 5) or from fac (combo 7, written by
// the DSCAL iteration of the same column).  Short columns (<= WB entries)
// keep their rows and sums in thread-local arrays and load each column j's
// tail in one batch of independent loads before merging it, so a column costs
// a few L2 round trips per predecessor rather than one per entry.
constexpr int WB = 32;

__device__ void ic0_col(int k, const ExecArgs& A, bool from_fac, int kernel) {
  const int c0 = __ldg(A.lc_ptr + k), c1 = __ldg(A.lc_ptr + k + 1);
  const int m = c1 - c0;
  const bool local = m <= WB;
  int rows[WB];
  double accl[WB];
  double* acc = local ? accl : A.work + c0;
  for (int a = 0; a < m; ++a) {
    if (local)
      rows[a] = __ldg(A.lc_idx + c0 + a);
    acc[a] = from_fac ? ld_cg(A.fac + c0 + a) : __ldg(A.lc_val + c0 + a);
  }
#define ROW(a) (local ? rows[(a)] : __ldg(A.lc_idx + c0 + (a)))
  for (int q = __ldg(A.rv_ptr + k); q < __ldg(A.rv_ptr + k + 1); ++q) {
    const int j = __ldg(A.rv_col + q);
    const int pj = __ldg(A.rv_pos + q);
    const int pe = __ldg(A.lc_ptr + j + 1);
    const double lkj = ld_cg(A.fac + pj);
    int a = 0;
    if (local && pe - pj <= WB) {
      int tr[WB];
      double tv[WB];
      for (int u = 0; u < pe - pj; ++u) {
        tr[u] = __ldg(A.lc_idx + pj + u);
        tv[u] = ld_cg(A.fac + pj + u);
      }
      for (int u = 0; u < pe - pj; ++u) {
        while (a < m && rows[a] < tr[u])
          ++a;
        if (a == m)
          break;
        if (rows[a] == tr[u])
          acc[a] = fsub_mul(acc[a], lkj, tv[u]);
      }
      continue;
    }
    for (int p = pj; p < pe; ++p) {
      const int i = __ldg(A.lc_idx + p);
      while (a < m && ROW(a) < i)
        ++a;
      if (a == m)
        break;
      if (ROW(a) == i)
        acc[a] = fsub_mul(acc[a], lkj, ld_cg(A.fac + p));
    }
  }
#undef ROW
  const double d = acc[0];
  if (d <= 0.0)
    report_error(A.err, kernel, k, k);
  const double lkk = __dsqrt_rn(d);
  A.fac[c0] = lkk;
  for (int a = 1; a < m; ++a)
    A.fac[c0 + a] = __ddiv_rn(acc[a], lkk);
}

// ilu0_row (kernels.hpp:246-272) by merging row i with the pivot rows' upper
// parts; initial values from ar_val (combo 6) or fac (combo 3, DSCAL'd).
// Short rows keep columns and sums in thread-local arrays and load each
// pivot row's upper part in one batch before merging it.
__device__ void ilu0_row(int i, const ExecArgs& A, bool from_fac, int kernel) {
  const int r0 = __ldg(A.ar_ptr + i), r1 = __ldg(A.ar_ptr + i + 1);
  const int m = r1 - r0;
  const bool local = m <= WB;
  int cols[WB];
  double accl[WB];
  double* acc = local ? accl : A.work + r0;
  for (int a = 0; a < m; ++a) {
    if (local)
      cols[a] = __ldg(A.ar_idx + r0 + a);
    acc[a] = from_fac ? ld_cg(A.fac + r0 + a) : __ldg(A.ar_val + r0 + a);
  }
#define COL(a) (local ? cols[(a)] : __ldg(A.ar_idx + r0 + (a)))
  for (int a = 0; a < m; ++a) {
    const int k = COL(a);
    if (k >= i)
      break;
    const int dk = __ldg(A.diag + k);
    const double piv = dk >= 0 ? ld_cg(A.fac + dk) : 0.0;
    if (dk < 0 || piv == 0.0)
      report_error(A.err, kernel, i, k);
    const double lik = __ddiv_rn(acc[a], piv);
    acc[a] = lik;
    if (dk < 0)
      continue;
    const int qe = __ldg(A.ar_ptr + k + 1);
    int b = a + 1;
    if (local && qe - dk - 1 <= WB) {
      int tc[WB];
      double tv[WB];
      for (int u = 0; u < qe - dk - 1; ++u) {
        tc[u] = __ldg(A.ar_idx + dk + 1 + u);
        tv[u] = ld_cg(A.fac + dk + 1 + u);
      }
      for (int u = 0; u < qe - dk - 1; ++u) {
        while (b < m && cols[b] < tc[u])
          ++b;
        if (b == m)
          break;
        if (cols[b] == tc[u])
          acc[b] = fsub_mul(acc[b], lik, tv[u]);
      }
      continue;
    }
    for (int q = dk + 1; q < qe; ++q) {
      const int j = __ldg(A.ar_idx + q);
      while (b < m && COL(b) < j)
        ++b;
      if (b == m)
        break;
      if (COL(b) == j)
        acc[b] = fsub_mul(acc[b], lik, ld_cg(A.fac + q));
    }
  }
#undef COL
  for (int a = 0; a < m; ++a)
    A.fac[r0 + a] = acc[a];
}

// run_iteration (kernels.hpp:508-570) for one (tag, iteration, system)
template <int COMBO>
__device__ void run_entry(int tag, int i, int s, const WaveArgs& W) {
  const ExecArgs& A = W.a;
  const int S = A.nsys;
  const size_t is = (size_t)i * S + s;
  switch (COMBO) {
  case 1:
    if (tag == 1)
      trsv_row(i, s, S, A.lr_ptr, A.lr_idx, A.lr_val, __ldg(A.vin + is), A.vmid, A.err, 1, i);
    else
      trsv_row(i, s, S, A.lr_ptr, A.lr_idx, A.lr_val, ld_cg(A.vmid + is), A.vout, A.err, 2, i);
    return;
  case 2:
    if (tag == 1) { // spmv_csr_row (kernels.hpp:152-158)
      double acc = 0.0;
      for (int p = __ldg(A.ar_ptr + i); p < __ldg(A.ar_ptr + i + 1); ++p)
        acc = __dadd_rn(acc, __dmul_rn(__ldg(A.ar_val + p), __ldg(A.vin + __ldg(A.ar_idx + p))));
      A.vmid[i] = acc;
    } else {
      trsv_row(i, s, S, A.lr_ptr, A.lr_idx, A.lr_val, ld_cg(A.vmid + is), A.vout, A.err, 2, i);
    }
    return;
  case 3:
    if (tag == 1) { // dscal_csr_row (kernels.hpp:274-279)
      const double di = __ldg(A.dvec + i);
      for (int p = __ldg(A.ar_ptr + i); p < __ldg(A.ar_ptr + i + 1); ++p)
        A.fac[p] = __dmul_rn(__dmul_rn(di, __ldg(A.ar_val + p)), __ldg(A.dvec + __ldg(A.ar_idx + p)));
    } else {
      ilu0_row(i, A, true, 2);
    }
    return;
  case 4:
    if (tag == 1) {
      trsv_row(i, s, S, A.lr_ptr, A.lr_idx, A.lr_val, __ldg(A.vin + is), A.vmid, A.err, 1, i);
    } else { // spmv_csc_col (kernels.hpp:162-168): atomic scatter, any order
      const double xj = ld_cg(A.vmid + i);
      for (int p = __ldg(W.m_ptr + i); p < __ldg(W.m_ptr + i + 1); ++p)
        atomicAdd(A.vout + __ldg(W.m_idx + p), __dmul_rn(__ldg(W.m_val + p), xj));
    }
    return;
  case 5:
    if (tag == 1) {
      ic0_col(i, A, false, 1);
    } else { // trsv_csc_row (kernels.hpp:200-210)
      double acc = __ldg(A.vin + i);
      for (int q = __ldg(A.rv_ptr + i); q < __ldg(A.rv_ptr + i + 1); ++q)
        acc = fsub_mul(acc, ld_cg(A.fac + __ldg(A.rv_pos + q)), ld_cg(A.vout + __ldg(A.rv_col + q)));
      const double d = ld_cg(A.fac + __ldg(A.lc_ptr + i));
      if (d == 0.0)
        report_error(A.err, 2, i, i);
      A.vout[i] = __ddiv_rn(acc, d);
    }
    return;
  case 6:
    if (tag == 1) {
      ilu0_row(i, A, false, 1);
    } else { // trsv_csr_unit_row (kernels.hpp:184-196)
      double acc = __ldg(A.vin + i);
      const int dp = __ldg(A.diag + i);
      const int end = dp >= 0 ? dp : __ldg(A.ar_ptr + i + 1);
      for (int p = __ldg(A.ar_ptr + i); p < end; ++p) {
        const int j = __ldg(A.ar_idx + p);
        if (j >= i)
          break;
        acc = fsub_mul(acc, ld_cg(A.fac + p), ld_cg(A.vout + j));
      }
      A.vout[i] = acc;
    }
    return;
  case 7:
    if (tag == 1) { // dscal_csc_col (kernels.hpp:281-286)
      const double dj = __ldg(A.dvec + i);
      for (int p = __ldg(A.lc_ptr + i); p < __ldg(A.lc_ptr + i + 1); ++p)
        A.fac[p] = __dmul_rn(__dmul_rn(__ldg(A.dvec + __ldg(A.lc_idx + p)), __ldg(A.lc_val + p)), dj);
    } else {
      ic0_col(i, A, true, 2);
    }
    return;
  case 8:
    if (tag == 1) {
      trsv_row(i, s, S, A.lr_ptr, A.lr_idx, A.lr_val, __ldg(A.vin + is), A.vmid, A.err, 1, i);
    } else { // backward iteration i = row n-1-i of L' (descending solve order)
      const int r = A.n - 1 - i;
      trsv_row(r, s, S, A.lt_ptr, A.lt_idx, A.lt_val, ld_cg(A.vmid + (size_t)r * S + s), A.vout,
               A.err, 2, i);
    }
    return;
  }
}

template <int COMBO>
__global__ void __launch_bounds__(kBlock) k_wavefront(const WaveArgs W) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const int S = W.a.nsys;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  for (int l = 0; l < W.nlev; ++l) {
    const int64_t b = __ldg(W.lptr + l), e = __ldg(W.lptr + l + 1);
    const int64_t work = (e - b) * S;
    for (int64_t w = tid; w < work; w += nth) {
      const int v = __ldg(W.verts + b + w / S);
      const int s = (int)(w % S);
      if (v < W.a.n)
        run_entry<COMBO>(1, v, s, W);
      else
        run_entry<COMBO>(2, v - W.a.n, s, W);
    }
    grid.sync(); // the barrier between s-partitions (SpinBarrier, executor.hpp:36-68)
  }
}

// run_sequential_reference (kernels.hpp:574-582) on one thread: every
// kernel-1 iteration ascending, then every kernel-2 iteration (the
// reference's sequential baseline, execute_sequential executor.hpp:315-322).
template <int COMBO> __global__ void k_sequential(const WaveArgs W) {
  const int S = W.a.nsys;
  for (int tag = 1; tag <= 2; ++tag)
    for (int i = 0; i < W.a.n; ++i)
      for (int s = 0; s < S; ++s)
        run_entry<COMBO>(tag, i, s, W);
}

template <int COMBO> void launch(const WaveArgs& w, cudaStream_t s) {
  if (w.nlev < 0) { // sequential
    k_sequential<COMBO><<<1, 1, 0, s>>>(w);
    count_launch();
    SFG_CUDA(cudaGetLastError());
    return;
  }
  auto kern = k_wavefront<COMBO>;
  int per_sm = 0;
  SFG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBlock, 0));
  if (per_sm < 1)
    per_sm = 1;
  const unsigned grid = (unsigned)(per_sm * sm_count());
  void* args[] = {(void*)&w};
  SFG_CUDA(cudaLaunchCooperativeKernel((const void*)kern, grid, kBlock, args, 0, s));
  count_launch();
}

__global__ void sched_pos_kernel(const uint8_t* __restrict__ tags, const int32_t* __restrict__ iters,
                                 int64_t ne, int32_t n, int64_t* pos, unsigned long long* bad) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < ne;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int tg = tags[q], it = iters[q];
    if ((tg != 1 && tg != 2) || it < 0 || it >= n) {
      atomicAdd(bad, 1ull);
      continue;
    }
    const int64_t v = (tg == 1 ? 0 : n) + it;
    if (atomicCAS(reinterpret_cast<unsigned long long*>(pos + v), ~0ull, (unsigned long long)q) != ~0ull)
      atomicAdd(bad, 1ull); // iteration scheduled twice
  }
}

__global__ void sched_edge_kernel(const int32_t* __restrict__ ptr, const int32_t* __restrict__ succ,
                                  int32_t nv, const int64_t* __restrict__ pos,
                                  unsigned long long* bad) {
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < nv;
       u += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pu = pos[u];
    if (pu == -1) {
      atomicAdd(bad, 1ull); // iteration never scheduled
      continue;
    }
    for (int e = ptr[u]; e < ptr[u + 1]; ++e) {
      const int64_t pv = pos[succ[e]];
      if (pv != -1 && pv < pu)
        atomicAdd(bad, 1ull);
    }
  }
}

} // namespace

int64_t check_schedule_order(const int32_t* jptr, const int32_t* jsucc, int32_t n,
                             const uint8_t* tags_h, const int32_t* iters_h, int64_t ne,
                             cudaStream_t s) {
  const int32_t nv = 2 * n;
  DBuf<int64_t> pos(nv > 0 ? nv : 1);
  DBuf<unsigned long long> bad(1);
  DBuf<uint8_t> tg(ne > 0 ? ne : 1);
  DBuf<int32_t> it(ne > 0 ? ne : 1);
  SFG_CUDA(cudaMemsetAsync(pos.p, 0xFF, sizeof(int64_t) * (size_t)(nv > 0 ? nv : 1), s));
  SFG_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(unsigned long long), s));
  if (ne > 0) {
    SFG_CUDA(cudaMemcpyAsync(tg.p, tags_h, (size_t)ne, cudaMemcpyHostToDevice, s));
    SFG_CUDA(cudaMemcpyAsync(it.p, iters_h, sizeof(int32_t) * (size_t)ne, cudaMemcpyHostToDevice, s));
    sched_pos_kernel<<<(unsigned)std::min<int64_t>((ne + 255) / 256, 4096), 256, 0, s>>>(
        tg.p, it.p, ne, n, pos.p, bad.p);
    count_launch();
  }
  if (nv > 0) {
    sched_edge_kernel<<<(unsigned)std::min<int64_t>((nv + 255) / 256, 4096), 256, 0, s>>>(
        jptr, jsucc, nv, pos.p, bad.p);
    count_launch();
  }
  unsigned long long h = 0;
  SFG_CUDA(cudaMemcpyAsync(&h, bad.p, sizeof(h), cudaMemcpyDeviceToHost, s));
  SFG_CUDA(cudaStreamSynchronize(s));
  return (int64_t)h + (ne != nv ? 1 : 0);
}

void launch_wavefront(const ExecArgs& a, int combo, const int32_t* verts, const int64_t* lptr,
                      int32_t nlev, const int32_t* m_ptr, const int32_t* m_idx,
                      const double* m_val, cudaStream_t s) {
  if (nlev == 0)
    return;
  WaveArgs w;
  w.a = a;
  w.combo = combo;
  w.verts = verts;
  w.lptr = lptr;
  w.nlev = nlev;
  w.m_ptr = m_ptr;
  w.m_idx = m_idx;
  w.m_val = m_val;
  switch (combo) {
  case 1:
    launch<1>(w, s);
    break;
  case 2:
    launch<2>(w, s);
    break;
  case 3:
    launch<3>(w, s);
    break;
  case 4:
    launch<4>(w, s);
    break;
  case 5:
    launch<5>(w, s);
    break;
  case 6:
    launch<6>(w, s);
    break;
  case 7:
    launch<7>(w, s);
    break;
  case 8:
    launch<8>(w, s);
    break;
  default:
    throw InvalidArgument("launch_wavefront: bad combo");
  }
}

} // namespace sfg
