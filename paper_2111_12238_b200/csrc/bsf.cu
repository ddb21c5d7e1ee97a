// bsf.cu -- blocked sync-free triangular-solve executor (see bsf.cuh).
//
// Kernel anatomy (one persistent CTA per SM, 256 threads):
//   * thread = (row slot, system): S systems of a row are S adjacent lanes,
//     so each nonzero's values for all systems are one contiguous load and
//     each x_j gather fetches all systems' x_j at once;
//   * a CTA claims the next block ticket, sets its shared-memory x cache of
//     the block to SENT, and its 256/S row slots walk the block's rows in
//     block-local wavefront order (slot k takes rows k, k+RS, ...);
//   * a row's in-block dependencies are polled in shared memory, the
//     external ones in global memory; the next row's indices, values and
//     external x words are loaded before the current row starts waiting
//     (software pipelining), so only the true dependency latency remains on
//     the critical path;
//   * the result goes to shared memory (for the block) and to global memory
//     (for later blocks and the output).
// Arithmetic is the reference's: ascending (forward) / descending (backward)
// storage order, separately rounded multiply and subtract, IEEE division.
#include "bsf.cuh"
#include "common.cuh"

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>

namespace sfg {

namespace {

constexpr int kThreads = 256;

template <typename T> struct TmpBuf {
  T* p = nullptr;
  cudaStream_t s;
  TmpBuf(int64_t n, cudaStream_t st) : s(st) {
    if (n > 0)
      SFG_CUDA(cudaMallocAsync(&p, sizeof(T) * (size_t)n, s));
  }
  ~TmpBuf() {
    if (p)
      cudaFreeAsync(p, s);
  }
};

inline unsigned grid_for(int64_t work, int block = 256) {
  int64_t g = (work + block - 1) / block;
  const int64_t cap = (int64_t)sm_count() * 32;
  if (g > cap)
    g = cap;
  return (unsigned)(g < 1 ? 1 : g);
}

// ---------------------------------------------------------------------------
// layout builder
// ---------------------------------------------------------------------------

// Block-local wavefront of every position: 1 + max over dependencies that
// fall into the same block (external ones count as already done).  Sync-free
// over ascending position tickets, like levels_kernel.
__global__ void local_levels_kernel(const int32_t* __restrict__ ptr,
                                    const int32_t* __restrict__ idx, int32_t n, int dir,
                                    int32_t B, int* level_pos, unsigned long long* counter) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    const long long base = claim_tickets(counter, 32);
    if (base >= n)
      break;
    const long long t = base + lane;
    if (t >= n)
      continue;
    const int r = dir > 0 ? (int)t : n - 1 - (int)t;
    const int blk = (int)(t / B);
    int lv = 1;
    const int e = __ldg(ptr + r + 1) - 1; // diagonal last
    for (int p = __ldg(ptr + r); p < e; ++p) {
      const int j = __ldg(idx + p);
      const int pj = dir > 0 ? j : n - 1 - j;
      if (pj / B == blk) {
        const int l = poll_pos_i32(level_pos + pj) + 1;
        lv = l > lv ? l : lv;
      }
    }
    st_relaxed_i32(level_pos + t, lv);
  }
}

__global__ void bsf_keys_kernel(const int* __restrict__ level_pos, int32_t n, int32_t B,
                                uint32_t* __restrict__ keys, int32_t* __restrict__ vals) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    keys[t] = (uint32_t)(t / B) * (uint32_t)(B + 1) + (uint32_t)level_pos[t];
    vals[t] = (int32_t)t;
  }
}

__global__ void bsf_slots_kernel(const int32_t* __restrict__ sorted_pos, int32_t n, int dir,
                                 const int32_t* __restrict__ ptr, int32_t* __restrict__ rowP,
                                 int32_t* __restrict__ slot_of, int32_t* __restrict__ cnt) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q <= n;
       q += (int64_t)gridDim.x * blockDim.x) {
    if (q == n) {
      cnt[n] = 0;
      continue;
    }
    const int t = sorted_pos[q];
    const int r = dir > 0 ? t : n - 1 - t;
    rowP[q] = r;
    slot_of[r] = (int32_t)q;
    cnt[q] = ptr[r + 1] - ptr[r] - 1;
  }
}

__global__ void bsf_fill_kernel(const int32_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                                const double* __restrict__ val, int32_t n, int32_t S, int dir,
                                int32_t B, const int32_t* __restrict__ rowP,
                                const int32_t* __restrict__ slot_of,
                                const int32_t* __restrict__ nptr, int32_t* __restrict__ nidx,
                                double* __restrict__ nval, double* __restrict__ dval) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int r = rowP[q];
    const int blk = (int)(q / B);
    const int b0 = ptr[r], e = ptr[r + 1] - 1;
    int w = nptr[q];
    for (int p = b0; p < e; ++p, ++w) {
      const int j = idx[p];
      const int pj = dir > 0 ? j : n - 1 - j;
      nidx[w] = (pj / B == blk) ? -(slot_of[j] - blk * B + 1) : j;
      for (int s = 0; s < S; ++s)
        nval[(int64_t)w * S + s] = val[(int64_t)p * S + s];
    }
    for (int s = 0; s < S; ++s)
      dval[q * S + s] = val[(int64_t)e * S + s];
  }
}

// batch starts: a new block-local wavefront, or every R-th slot inside one
__global__ void bsf_runstart_kernel(const uint32_t* __restrict__ skeys, int32_t n,
                                    int32_t* __restrict__ rs) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x)
    rs[q] = (q == 0 || skeys[q] != skeys[q - 1]) ? (int32_t)q : 0;
}

__global__ void bsf_batchflag_kernel(const int32_t* __restrict__ run_start, int32_t n, int32_t R,
                                     int32_t* __restrict__ flag) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q <= n;
       q += (int64_t)gridDim.x * blockDim.x)
    flag[q] = q == n ? 0 : (((int32_t)q - run_start[q]) % R == 0 ? 1 : 0);
}

__global__ void bsf_bptr_kernel(const int32_t* __restrict__ flag, const int32_t* __restrict__ bid,
                                int32_t n, int32_t B, int32_t nblk, int32_t nbatch,
                                int32_t* __restrict__ bptr, int32_t* __restrict__ blk_batch) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q <= n;
       q += (int64_t)gridDim.x * blockDim.x) {
    if (q == n) {
      bptr[nbatch] = n;
      blk_batch[nblk] = nbatch;
      continue;
    }
    if (flag[q])
      bptr[bid[q]] = (int32_t)q;
    if (q % B == 0)
      blk_batch[q / B] = bid[q];
  }
}

int bits_for(int64_t maxval) {
  int b = 1;
  while (b < 62 && (1ll << b) <= maxval)
    ++b;
  return b;
}

// ---------------------------------------------------------------------------
// executor
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long ld_shared_volatile(const unsigned long long* p) {
  return *reinterpret_cast<const volatile unsigned long long*>(p);
}
__device__ __forceinline__ void st_shared_volatile(unsigned long long* p, unsigned long long v) {
  *reinterpret_cast<volatile unsigned long long*>(p) = v;
}
__device__ __forceinline__ double poll_shared(const unsigned long long* p) {
  unsigned long long v = ld_shared_volatile(p);
  while (v == SENT)
    v = ld_shared_volatile(p);
  return __longlong_as_double((long long)v);
}
__device__ __forceinline__ unsigned long long canon(double x) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return b == SENT ? CANON_NAN : b;
}

// One row of a solve as staged by the software pipeline.
template <int CH> struct Row {
  int row, e0, cnt;
  int code[CH];
  double v[CH];
  unsigned long long xe[CH]; // external x words loaded ahead (SENT if not ready)
  double d;
  unsigned long long rhs;
};

template <int S, int CH>
__device__ __forceinline__ void stage_row(Row<CH>& R, int q, const int32_t* __restrict__ rowP,
                                          const int32_t* __restrict__ nptr,
                                          const int32_t* __restrict__ nidx,
                                          const double* __restrict__ nval,
                                          const double* __restrict__ dval, const double* x,
                                          const double* rhs_vec, bool rhs_polled, int s) {
  R.row = __ldg(rowP + q);
  R.e0 = __ldg(nptr + q);
  R.cnt = __ldg(nptr + q + 1) - R.e0;
  R.d = __ldg(dval + (size_t)q * S + s);
#pragma unroll
  for (int a = 0; a < CH; ++a)
    if (a < R.cnt) {
      R.code[a] = __ldg(nidx + R.e0 + a);
      R.v[a] = __ldg(nval + (size_t)(R.e0 + a) * S + s);
    }
#pragma unroll
  for (int a = 0; a < CH; ++a)
    if (a < R.cnt)
      R.xe[a] = R.code[a] >= 0 ? ld_relaxed_u64(x + (size_t)R.code[a] * S + s) : SENT;
  if (rhs_vec)
    R.rhs = rhs_polled
                ? ld_relaxed_u64(rhs_vec + (size_t)R.row * S + s)
                : (unsigned long long)__double_as_longlong(__ldg(rhs_vec + (size_t)R.row * S + s));
}

// acc = rhs - sum v * x over the row; in-block x from the shared cache,
// external x from the staged words (re-polled while SENT).
template <int S, int CH>
__device__ __forceinline__ double solve_staged(const Row<CH>& R, double rhs,
                                               const unsigned long long* cache, const double* x,
                                               const int32_t* __restrict__ nidx,
                                               const double* __restrict__ nval, int s) {
  double acc = rhs;
#pragma unroll
  for (int a = 0; a < CH; ++a)
    if (a < R.cnt) {
      const int c = R.code[a];
      double xj;
      if (c < 0)
        xj = poll_shared(cache + (size_t)(-c - 1) * S + s);
      else
        xj = R.xe[a] != SENT ? __longlong_as_double((long long)R.xe[a])
                             : poll_f64(x + (size_t)c * S + s, 0);
      acc = __dsub_rn(acc, __dmul_rn(R.v[a], xj));
    }
  for (int a = CH; a < R.cnt; ++a) { // rows longer than the staging width
    const int c = __ldg(nidx + R.e0 + a);
    const double v = __ldg(nval + (size_t)(R.e0 + a) * S + s);
    const double xj = c < 0 ? poll_shared(cache + (size_t)(-c - 1) * S + s)
                            : poll_f64(x + (size_t)c * S + s, 0);
    acc = __dsub_rn(acc, __dmul_rn(v, xj));
  }
  return acc;
}

// Second solve of combo 1 on the same row (x2 = inv(L) z): its external x2
// words are not staged (they live in another vector).
template <int S, int CH>
__device__ __forceinline__ double solve_second(const Row<CH>& R, double rhs,
                                               const unsigned long long* cache, const double* x,
                                               const int32_t* __restrict__ nidx,
                                               const double* __restrict__ nval, int s) {
  double acc = rhs;
  unsigned long long xe[CH];
#pragma unroll
  for (int a = 0; a < CH; ++a)
    if (a < R.cnt)
      xe[a] = R.code[a] >= 0 ? ld_relaxed_u64(x + (size_t)R.code[a] * S + s) : SENT;
#pragma unroll
  for (int a = 0; a < CH; ++a)
    if (a < R.cnt) {
      const int c = R.code[a];
      double xj;
      if (c < 0)
        xj = poll_shared(cache + (size_t)(-c - 1) * S + s);
      else
        xj = xe[a] != SENT ? __longlong_as_double((long long)xe[a])
                           : poll_f64(x + (size_t)c * S + s, 0);
      acc = __dsub_rn(acc, __dmul_rn(R.v[a], xj));
    }
  for (int a = CH; a < R.cnt; ++a) {
    const int c = __ldg(nidx + R.e0 + a);
    const double v = __ldg(nval + (size_t)(R.e0 + a) * S + s);
    const double xj = c < 0 ? poll_shared(cache + (size_t)(-c - 1) * S + s)
                            : poll_f64(x + (size_t)c * S + s, 0);
    acc = __dsub_rn(acc, __dmul_rn(v, xj));
  }
  return acc;
}

template <int S, int CH, int COMBO>
__global__ void __launch_bounds__(kThreads, 1) k_bsf(const BsfArgs A) {
  extern __shared__ unsigned long long cache[];
  __shared__ long long s_ticket;
  constexpr int W = kThreads / 32;
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int g = (tid & 31) / S; // slot within a batch
  const int s = tid % S;
  const int maxB = A.Bf > A.Bb ? A.Bf : A.Bb;
  unsigned long long* cache2 = cache + (size_t)maxB * S; // combo 1 second solve
  for (;;) {
    if (tid == 0)
      s_ticket = (long long)atomicAdd(A.counter, 1ull);
    __syncthreads();
    const long long ti = s_ticket;
    if (ti >= A.nt)
      break;
    const int32_t tk = __ldg(A.tickets + ti);
    const int kind = tk >> 28;
    const int bi = tk & 0x0FFFFFFF;
    if (COMBO == 4 && kind == TK_Y) {
      // SpMV rows of block bi: row gather in the sequential CSC scatter's
      // order (see executor.cu gather_row), x polled in global memory.
      const int r0 = bi * A.By;
      const int r1 = min(A.n, r0 + A.By);
      for (int r = r0 + tid; r < r1; r += kThreads) {
        double acc = 0.0;
        for (int p = __ldg(A.ar_ptr + r); p < __ldg(A.ar_ptr + r + 1); ++p)
          acc = __dadd_rn(acc, __dmul_rn(__ldg(A.ar_val + p),
                                         poll_f64(A.vmid + __ldg(A.ar_idx + p), 0)));
        A.vout[r] = acc;
      }
    } else {
      const bool bwd = kind == TK_BWD;
      const int B = bwd ? A.Bb : A.Bf;
      const int32_t* rowP = bwd ? A.b_rowP : A.f_rowP;
      const int32_t* nptr = bwd ? A.b_ptr : A.f_ptr;
      const int32_t* nidx = bwd ? A.b_idx : A.f_idx;
      const double* nval = bwd ? A.b_val : A.f_val;
      const double* dval = bwd ? A.b_diag : A.f_diag;
      const int q0 = bi * B;
      const int q1 = min(A.n, q0 + B);
      const int ncache = COMBO == 1 ? 2 : 1;
      for (int i = tid; i < (q1 - q0) * S; i += kThreads) {
        cache[i] = SENT;
        if (ncache == 2)
          cache2[i] = SENT;
      }
      __syncthreads();
      // which vectors this block reads / writes
      const bool first = COMBO == 1 ? (A.phase & 1) != 0 : true;
      const bool second = COMBO == 1 && (A.phase & 2);
      double* xout = bwd ? A.vout : A.vmid;
      const double* rhs_vec = bwd ? A.vmid : A.vin;
      const bool rhs_polled = bwd;
      const int kernel = bwd ? 2 : 1;
      // warp w walks batches bb0 + w, bb0 + w + W, ...; lane group g takes
      // the g-th slot of a batch (all slots of a batch share one wavefront)
      const int32_t* bptr = bwd ? A.b_bptr : A.f_bptr;
      const int32_t* blkb = bwd ? A.b_blkb : A.f_blkb;
      const int bb1 = __ldg(blkb + bi + 1);
      int bat = __ldg(blkb + bi) + warp;
      int q = -1;
      Row<CH> cur;
      bool have = false;
      auto slot_of_batch = [&](int b) {
        const int qq = __ldg(bptr + b) + g;
        return qq < __ldg(bptr + b + 1) ? qq : -1;
      };
      if (bat < bb1) {
        q = slot_of_batch(bat);
        have = true;
        if (q >= 0)
          stage_row<S, CH>(cur, q, rowP, nptr, nidx, nval, dval, xout,
                           first ? rhs_vec : A.vmid, first ? rhs_polled : true, s);
      }
      while (have) {
        const int batn = bat + W;
        const bool hn = batn < bb1;
        int qn = -1;
        Row<CH> nxt;
        if (hn) {
          qn = slot_of_batch(batn);
          if (qn >= 0)
            stage_row<S, CH>(nxt, qn, rowP, nptr, nidx, nval, dval, xout,
                             first ? rhs_vec : A.vmid, first ? rhs_polled : true, s);
        }
        if (q >= 0) {
          const int r = cur.row;
          const int seq = bwd ? A.n - 1 - r : r;
          double z;
          if (first) {
            const double rhs = cur.rhs != SENT ? __longlong_as_double((long long)cur.rhs)
                                               : poll_f64(rhs_vec + (size_t)r * S + s, 0);
            const double acc = solve_staged<S, CH>(cur, rhs, cache, xout, nidx, nval, s);
            if (cur.d == 0.0)
              report_error(A.err, kernel, seq, r);
            z = __ddiv_rn(acc, cur.d);
            const unsigned long long zb = canon(z);
            st_shared_volatile(cache + (size_t)(q - q0) * S + s, zb);
            st_relaxed_u64(xout + (size_t)r * S + s, zb);
          } else {
            z = cur.rhs != SENT ? __longlong_as_double((long long)cur.rhs)
                                : poll_f64(A.vmid + (size_t)r * S + s, 0);
          }
          if (second) {
            const double acc = solve_second<S, CH>(cur, z, cache2, A.vout, nidx, nval, s);
            if (cur.d == 0.0)
              report_error(A.err, 2, r, r);
            const unsigned long long xb = canon(__ddiv_rn(acc, cur.d));
            st_shared_volatile(cache2 + (size_t)(q - q0) * S + s, xb);
            st_relaxed_u64(A.vout + (size_t)r * S + s, xb);
          }
        }
        cur = nxt;
        q = qn;
        bat = batn;
        have = hn;
      }
    }
    __syncthreads();
  }
}

template <int S, int CH, int COMBO> void launch_t(const BsfArgs& a, cudaStream_t s) {
  const int maxB = std::max(a.Bf, a.Bb);
  const size_t smem = (size_t)(COMBO == 1 ? 2 : 1) * maxB * S * sizeof(unsigned long long);
  if (smem > 200 * 1024)
    throw InvalidArgument("BSF block too large for shared memory (lower SFG_BSF_B)");
  auto kern = k_bsf<S, CH, COMBO>;
  SFG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  SFG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem));
  if (per_sm < 1)
    throw CudaError("k_bsf does not fit on an SM (block too large)");
  if (a.blocks_per_sm > 0 && a.blocks_per_sm < per_sm)
    per_sm = a.blocks_per_sm;
  int64_t grid = (int64_t)per_sm * sm_count();
  if (grid > a.nt)
    grid = a.nt;
  if (grid < 1)
    return;
  kern<<<(unsigned)grid, kThreads, smem, s>>>(a);
  count_launch();
  SFG_CUDA(cudaGetLastError());
}

template <int COMBO> void launch_c(const BsfArgs& a, cudaStream_t s) {
  switch (a.S) {
  case 1:
    launch_t<1, 8, COMBO>(a, s);
    break;
  case 2:
    launch_t<2, 16, COMBO>(a, s);
    break;
  case 4:
    launch_t<4, 16, COMBO>(a, s);
    break;
  case 8:
    launch_t<8, 16, COMBO>(a, s);
    break;
  case 16:
    launch_t<16, 16, COMBO>(a, s);
    break;
  case 32:
    launch_t<32, 16, COMBO>(a, s);
    break;
  default:
    throw InvalidArgument("nsys must be a power of two <= 32");
  }
}

} // namespace

void build_bsf(const int32_t* ptr, const int32_t* idx, const double* val, int32_t n, int32_t S,
               int dir, int32_t B, BsfLayout& out, cudaStream_t s) {
  out.n = n;
  out.S = S;
  out.B = B;
  out.dir = dir;
  out.nblk = (n + B - 1) / B;
  out.rowP.alloc(n > 0 ? n : 1);
  out.nptr.alloc((int64_t)n + 1);
  out.dval.alloc((int64_t)(n > 0 ? n : 1) * S);
  if (n == 0) {
    SFG_CUDA(cudaMemsetAsync(out.nptr.p, 0, sizeof(int32_t), s));
    out.nidx.alloc(1);
    out.nval.alloc(1);
    out.bptr.alloc(1);
    out.blk_batch.alloc(1);
    SFG_CUDA(cudaMemsetAsync(out.bptr.p, 0, sizeof(int32_t), s));
    SFG_CUDA(cudaMemsetAsync(out.blk_batch.p, 0, sizeof(int32_t), s));
    return;
  }
  TmpBuf<int> level(n, s);
  TmpBuf<unsigned long long> counter(1, s);
  SFG_CUDA(cudaMemsetAsync(level.p, 0, sizeof(int) * (size_t)n, s));
  SFG_CUDA(cudaMemsetAsync(counter.p, 0, sizeof(unsigned long long), s));
  {
    int per_sm = 0;
    SFG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, local_levels_kernel, 256, 0));
    int64_t blocks = ((int64_t)n + 255) / 256;
    const int64_t cap = (int64_t)(per_sm < 1 ? 1 : per_sm) * sm_count();
    if (blocks > cap)
      blocks = cap;
    local_levels_kernel<<<(unsigned)blocks, 256, 0, s>>>(ptr, idx, n, dir, B, level.p, counter.p);
    count_launch();
  }
  TmpBuf<uint32_t> keys(n, s), keys_out(n, s);
  TmpBuf<int32_t> vals(n, s), sorted(n, s);
  bsf_keys_kernel<<<grid_for(n), 256, 0, s>>>(level.p, n, B, keys.p, vals.p);
  count_launch();
  const int64_t maxkey = (int64_t)out.nblk * (B + 1);
  size_t bytes = 0;
  SFG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys.p, keys_out.p, vals.p, sorted.p,
                                           n, 0, bits_for(maxkey), s));
  {
    TmpBuf<char> tmp((int64_t)bytes, s);
    SFG_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, keys.p, keys_out.p, vals.p, sorted.p,
                                             n, 0, bits_for(maxkey), s));
  }
  {
    TmpBuf<int32_t> lmax(1, s);
    bytes = 0;
    SFG_CUDA(cub::DeviceReduce::Max(nullptr, bytes, level.p, lmax.p, n, s));
    TmpBuf<char> tmp((int64_t)bytes, s);
    SFG_CUDA(cub::DeviceReduce::Max(tmp.p, bytes, level.p, lmax.p, n, s));
    SFG_CUDA(cudaMemcpyAsync(&out.max_local_levels, lmax.p, sizeof(int32_t),
                             cudaMemcpyDeviceToHost, s));
  }
  {
    // batches of <= 32/S slots within one block-local wavefront
    const int32_t R = 32 / S > 0 ? 32 / S : 1;
    TmpBuf<int32_t> rstart(n, s), flag((int64_t)n + 1, s), bid((int64_t)n + 1, s);
    bsf_runstart_kernel<<<grid_for(n), 256, 0, s>>>(keys_out.p, n, rstart.p);
    size_t b2 = 0;
    SFG_CUDA(cub::DeviceScan::InclusiveScan(nullptr, b2, rstart.p, rstart.p, cub::Max(), n, s));
    {
      TmpBuf<char> tmp((int64_t)b2, s);
      SFG_CUDA(cub::DeviceScan::InclusiveScan(tmp.p, b2, rstart.p, rstart.p, cub::Max(), n, s));
    }
    bsf_batchflag_kernel<<<grid_for((int64_t)n + 1), 256, 0, s>>>(rstart.p, n, R, flag.p);
    b2 = 0;
    SFG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, b2, flag.p, bid.p, n + 1, s));
    {
      TmpBuf<char> tmp((int64_t)b2, s);
      SFG_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, b2, flag.p, bid.p, n + 1, s));
    }
    int32_t nb = 0;
    SFG_CUDA(cudaMemcpyAsync(&nb, bid.p + n, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    SFG_CUDA(cudaStreamSynchronize(s));
    out.nbatch = nb;
    out.bptr.alloc((int64_t)nb + 1);
    out.blk_batch.alloc((int64_t)out.nblk + 1);
    bsf_bptr_kernel<<<grid_for((int64_t)n + 1), 256, 0, s>>>(flag.p, bid.p, n, B, out.nblk, nb,
                                                             out.bptr.p, out.blk_batch.p);
    count_launch(3);
  }
  TmpBuf<int32_t> slot_of(n, s), cnt((int64_t)n + 1, s);
  bsf_slots_kernel<<<grid_for((int64_t)n + 1), 256, 0, s>>>(sorted.p, n, dir, ptr, out.rowP.p,
                                                            slot_of.p, cnt.p);
  count_launch();
  bytes = 0;
  SFG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, cnt.p, out.nptr.p, n + 1, s));
  {
    TmpBuf<char> tmp((int64_t)bytes, s);
    SFG_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, cnt.p, out.nptr.p, n + 1, s));
  }
  int32_t nent = 0;
  SFG_CUDA(cudaMemcpyAsync(&nent, out.nptr.p + n, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  SFG_CUDA(cudaStreamSynchronize(s));
  out.nent = nent;
  out.nidx.alloc(nent > 0 ? nent : 1);
  out.nval.alloc((int64_t)(nent > 0 ? nent : 1) * S);
  bsf_fill_kernel<<<grid_for(n), 256, 0, s>>>(ptr, idx, val, n, S, dir, B, out.rowP.p, slot_of.p,
                                              out.nptr.p, out.nidx.p, out.nval.p, out.dval.p);
  count_launch();
  SFG_CUDA(cudaGetLastError());
  SFG_CUDA(cudaStreamSynchronize(s));
}

std::vector<int32_t> bsf_tickets(int combo, const BsfLayout& fwd, const BsfLayout* bwd,
                                 int32_t y_blocks, const std::vector<int32_t>& y_after,
                                 int64_t* k1_count) {
  std::vector<int32_t> t;
  if (combo == 4) {
    // y block k goes right after the forward block it last reads
    std::vector<std::vector<int32_t>> after((size_t)fwd.nblk);
    std::vector<int32_t> first;
    for (int32_t k = 0; k < y_blocks; ++k) {
      const int32_t b = y_after[(size_t)k];
      if (b < 0)
        first.push_back(k);
      else
        after[(size_t)std::min(b, fwd.nblk - 1)].push_back(k);
    }
    for (int32_t k : first)
      t.push_back(ticket(TK_Y, k));
    for (int32_t b = 0; b < fwd.nblk; ++b) {
      t.push_back(ticket(TK_FWD, b));
      for (int32_t k : after[(size_t)b])
        t.push_back(ticket(TK_Y, k));
    }
    *k1_count = fwd.nblk;
    return t;
  }
  for (int32_t b = 0; b < fwd.nblk; ++b)
    t.push_back(ticket(TK_FWD, b));
  *k1_count = fwd.nblk;
  if (combo == 8 && bwd)
    for (int32_t b = 0; b < bwd->nblk; ++b)
      t.push_back(ticket(TK_BWD, b));
  return t;
}

void launch_bsf(const BsfArgs& a, cudaStream_t s) {
  if (a.nt <= 0)
    return;
  switch (a.combo) {
  case 1:
    launch_c<1>(a, s);
    break;
  case 4:
    if (a.S != 1)
      throw InvalidArgument("combo 4 supports a single system");
    launch_t<1, 8, 4>(a, s);
    break;
  case 8:
    launch_c<8>(a, s);
    break;
  default:
    throw InvalidArgument("launch_bsf: bad combo");
  }
}

} // namespace sfg
