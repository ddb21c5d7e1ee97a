// ell.cu -- chain-ELL layout builder and the TMA-staged chain executor
// (see ell.cuh).
//
// Executor anatomy (one warp per chain, lane = (row-in-tile k, system s)):
//   iteration u waits on the mbarrier of iteration u-1, then issues, with
//   Blackwell's 1-D bulk copies (cp.async.bulk -> shared memory, completion
//   counted in bytes on a per-warp mbarrier):
//     * the dependency indices of tile u+2           (one copy)
//     * the values + carry + diagonal of tile u+1     (one copy)
//     * the right-hand sides of tile u+1             (one copy)
//     * the x row of every dependency of tile u+1   (one 8*S-byte copy each,
//       read through L2, so a word published by another SM is seen as soon
//       as it lands there; a word still SENT is re-polled)
//   and completes tile u from shared memory: all rows add their terms in
//   the reference order in parallel, then the carry runs through the G rows
//   with warp shuffles, dividing with a reciprocal computed off the chain.
#include "common.cuh"
#include "ell.cuh"

#include <cub/device/device_reduce.cuh>

namespace sfg {

namespace {

constexpr unsigned FULL = 0xffffffffu;

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

__device__ __forceinline__ bool chained_at(int p, const int32_t* __restrict__ chain_of,
                                           const int32_t* __restrict__ cstart) {
  return cstart[chain_of[p]] != p;
}

__global__ void ell_width_kernel(const int32_t* __restrict__ ptr, int32_t n, int dir,
                                 const int32_t* __restrict__ chain_of,
                                 const int32_t* __restrict__ cstart, int32_t* __restrict__ w) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int r = dir > 0 ? (int)p : n - 1 - (int)p;
    const int nd = ptr[r + 1] - ptr[r] - 1;
    w[p] = chained_at((int)p, chain_of, cstart) ? nd - 1 : nd;
  }
}

__global__ void ell_fill_kernel(const int32_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                                const double* __restrict__ val, int32_t n, int32_t S, int dir,
                                int32_t CHN, const int32_t* __restrict__ chain_of,
                                const int32_t* __restrict__ cstart, int32_t* __restrict__ eidx,
                                double* __restrict__ eval) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int r = dir > 0 ? (int)p : n - 1 - (int)p;
    const int b = ptr[r], e = ptr[r + 1] - 1;
    const bool ch = chained_at((int)p, chain_of, cstart);
    const int m = ch ? e - 1 - b : e - b;
    int32_t* ir = eidx + p * CHN;
    double* vr = eval + p * (int64_t)(CHN + 2) * S;
    for (int a = 0; a < CHN; ++a) {
      ir[a] = a < m ? idx[b + a] : n; // padding -> the all-zero row n
      for (int s = 0; s < S; ++s)
        vr[a * S + s] = a < m ? val[(int64_t)(b + a) * S + s] : 0.0;
    }
    for (int s = 0; s < S; ++s) {
      vr[CHN * S + s] = ch ? val[(int64_t)(e - 1) * S + s] : 0.0;
      vr[(CHN + 1) * S + s] = val[(int64_t)e * S + s];
    }
  }
}

// ---- PTX helpers: mbarrier + 1-D bulk copy ----------------------------------
__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
               "[%3];" ::"r"(smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}
__device__ __forceinline__ unsigned long long gtimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

template <int S, int G, int CHN> struct alignas(16) EllWarpBuf {
  double val[2][G][CHN + 2][S];
  double rhs[2][G][S];
  int32_t idx[3][G][CHN];
  unsigned long long bar[2];
};

template <int S, int G, int CHN>
__global__ void __launch_bounds__(160) k_chain_ell(const EllArgs A) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  using Buf = EllWarpBuf<S, G, CHN>;
  Buf& W = reinterpret_cast<Buf*>(smem_raw)[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  const int k = lane / S;
  const int s = lane % S;
  const bool lane_on = k < G;
  if (lane == 0) {
    mbar_init(&W.bar[0], 32);
    mbar_init(&W.bar[1], 32);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  unsigned phase[2] = {0u, 0u};
  const int total = A.seg_end - A.seg_begin;
  for (;;) {
    unsigned long long w0 = 0;
    if (lane == 0)
      w0 = atomicAdd(A.counter, 1ull);
    const long long wi = (long long)__shfl_sync(FULL, w0, 0);
    if (wi >= total)
      break;
    const int item = A.seg_begin + (int)wi;
    const bool bwd = item >= A.f_nbatch;
    const int bi = bwd ? item - A.f_nbatch : item;
    const int32_t* cstart = bwd ? A.b_cstart : A.f_cstart;
    const int32_t* corder = bwd ? A.b_corder : A.f_corder;
    const int32_t* bptr = bwd ? A.b_bptr : A.f_bptr;
    const int32_t* clev = bwd ? A.b_level : A.f_level;
    const int32_t* eidx = bwd ? A.b_eidx : A.f_eidx;
    const double* eval = bwd ? A.b_eval : A.f_eval;
    const int c = __ldg(corder + __ldg(bptr + bi));
    const int p0 = __ldg(cstart + c);
    const int len = __ldg(cstart + c + 1) - p0;
    const int skew = __ldg(clev + c) % G;
    const int ntiles = (len + skew + G - 1) / G;
    const int n = A.n;
    double* xo = bwd ? A.vout : A.vmid;
    const double* rv = bwd ? A.vmid : A.vin;
    const int kern = bwd ? 2 : 1;
    // first position of tile u (may lie before the chain start)
    auto tile_q0 = [&](int u) { return p0 + G * u - skew; };
    double carry = 0.0;
    unsigned long long xc[CHN], xn[CHN]; // x words of tiles u and u+1
#pragma unroll
    for (int a = 0; a < CHN; ++a)
      xc[a] = xn[a] = SENT;
#pragma unroll 1
    for (int u = -2; u < ntiles; ++u) {
      if (u >= -1) {
        mbar_wait(&W.bar[(u - 1) & 1], phase[(u - 1) & 1]);
        phase[(u - 1) & 1] ^= 1u;
      }
      // ---- issue tile u+2 indices and tile u+1 data on barrier u&1
      {
        unsigned long long* bar = &W.bar[u & 1];
        unsigned bytes = 0;
        fence_proxy_async();
        __syncwarp();
        const int ui = u + 2, ud = u + 1;
        if (lane == 0 && ui < ntiles) {
          const int q0 = tile_q0(ui);
          const int lo = max(q0, p0), hi = min(q0 + G, p0 + len);
          const unsigned nb = (unsigned)(hi - lo) * CHN * 4u;
          bulk_g2s(&W.idx[ui % 3][lo - q0][0], eidx + (size_t)lo * CHN, nb, bar);
          bytes += nb;
        }
        if (ud >= 0 && ud < ntiles) {
          const int q0 = tile_q0(ud);
          const int lo = max(q0, p0), hi = min(q0 + G, p0 + len);
          if (lane == 0) {
            const unsigned nv = (unsigned)(hi - lo) * (CHN + 2) * S * 8u;
            bulk_g2s(&W.val[ud & 1][lo - q0][0][0], eval + (size_t)lo * (CHN + 2) * S, nv, bar);
            const unsigned nr = (unsigned)(hi - lo) * S * 8u;
            if (!bwd) {
              bulk_g2s(&W.rhs[ud & 1][lo - q0][0], rv + (size_t)lo * S, nr, bar);
            } else {
              // rows n-1-q descend with q: memory rows [n-hi, n-lo) land
              // reversed; smem row j holds position hi-1-j
              bulk_g2s(&W.rhs[ud & 1][0][0], rv + (size_t)(n - hi) * S, nr, bar);
            }
            bytes += nv + nr;
          }
          // first (speculative) read of every x word tile u+1 needs, with
          // plain per-lane loads (indices arrived with the previous barrier)
          const int q = q0 + k;
          if (lane_on && q >= lo && q < hi) {
#pragma unroll
            for (int a = 0; a < CHN; ++a)
              xn[a] = ld_relaxed_u64(xo + (size_t)W.idx[ud % 3][k][a] * S + s);
          }
        }
        mbar_arrive_tx(bar, bytes);
      }
      // ---- complete tile u (tile-synchronous: all rows gather their terms,
      // then the carry runs through the tile)
      if (u >= 0) {
        const int q0 = tile_q0(u);
        const int q = q0 + k;
        const bool act = lane_on && q >= p0 && q < p0 + len;
        const int slot = u & 1;
        double acc = 0.0, d = 1.0, vc = 0.0, rd = 1.0;
        int r = 0;
        if (act) {
          r = bwd ? n - 1 - q : q;
          d = W.val[slot][k][CHN + 1][s];
          vc = W.val[slot][k][CHN][s];
          rd = __drcp_rn(d);
          const int hi = min(q0 + G, p0 + len);
          unsigned long long rw =
              (unsigned long long)__double_as_longlong(bwd ? W.rhs[slot][hi - 1 - q][s]
                                                           : W.rhs[slot][k][s]);
          if (bwd && is_sent_hi(rw))
            rw = (unsigned long long)__double_as_longlong(poll_f64(rv + (size_t)r * S + s, 0));
          acc = __longlong_as_double((long long)rw);
          for (;;) {
            bool pending = false;
#pragma unroll
            for (int a = 0; a < CHN; ++a)
              pending |= is_sent_hi(xc[a]);
            if (!pending)
              break;
#pragma unroll
            for (int a = 0; a < CHN; ++a)
              if (is_sent_hi(xc[a]))
                xc[a] = ld_relaxed_u64(xo + (size_t)W.idx[u % 3][k][a] * S + s);
          }
#pragma unroll
          for (int a = 0; a < CHN; ++a)
            acc = __dsub_rn(acc, __dmul_rn(W.val[slot][k][a][s],
                                           __longlong_as_double((long long)xc[a])));
          if (d == 0.0)
            report_error(A.err, kern, bwd ? n - 1 - r : r, r);
        }
        const bool chained = q > p0;
        double x = 0.0;
#pragma unroll
        for (int kk = 0; kk < G; ++kk) {
          const double v = chained ? __dsub_rn(acc, __dmul_rn(vc, carry)) : acc;
          const double q0d = __dmul_rn(v, rd);
          double qq = __fma_rn(__fma_rn(-q0d, d, v), rd, q0d);
          const bool mine = act && k == kk;
          if (__builtin_expect(mine && !(exp_in_safe_range(v) && exp_in_safe_range(d)), 0))
            qq = ieee_div_slow(v, d);
          if (mine) {
            x = qq;
            publish_f64(xo + (size_t)r * S + s, qq);
          }
          carry = __shfl_sync(FULL, x, kk * S + s);
        }
        if (A.trace && lane == 0 && u < A.trace_tiles)
          A.trace[(size_t)item * A.trace_tiles + u] = gtimer_ns();
      }
#pragma unroll
      for (int a = 0; a < CHN; ++a)
        xc[a] = xn[a];
    }
    // the last iteration armed barrier (ntiles-1)&1 with an empty issue
    mbar_wait(&W.bar[(ntiles - 1) & 1], phase[(ntiles - 1) & 1]);
    phase[(ntiles - 1) & 1] ^= 1u;
  }
}

template <int S, int CHN> void launch_s(const EllArgs& a, cudaStream_t s) {
  constexpr int G = 32 / S < 8 ? 32 / S : 8;
  using Buf = EllWarpBuf<S, G, CHN>;
  const int wpc = 5;
  const size_t smem = (size_t)wpc * sizeof(Buf);
  auto kern = k_chain_ell<S, G, CHN>;
  SFG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  SFG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * wpc, smem));
  if (per_sm < 1)
    throw CudaError("k_chain_ell does not fit on an SM");
  if (a.blocks_per_sm > 0 && a.blocks_per_sm < per_sm)
    per_sm = a.blocks_per_sm;
  const int64_t items = a.seg_end - a.seg_begin;
  int64_t grid = (items + wpc - 1) / wpc;
  if (grid > (int64_t)per_sm * sm_count())
    grid = (int64_t)per_sm * sm_count();
  if (grid < 1)
    return;
  kern<<<(unsigned)grid, 32 * wpc, smem, s>>>(a);
  count_launch();
  SFG_CUDA(cudaGetLastError());
}

template <int S> void launch_w(const EllArgs& a, int32_t CHN, cudaStream_t s) {
  switch (CHN) {
  case 4:
    launch_s<S, 4>(a, s);
    break;
  case 8:
    launch_s<S, 8>(a, s);
    break;
  case 12:
    launch_s<S, 12>(a, s);
    break;
  case 16:
    launch_s<S, 16>(a, s);
    break;
  default:
    throw InvalidArgument("chain-ELL width must be 4, 8, 12 or 16");
  }
}

} // namespace

int32_t ell_width(const int32_t* ptr, const int32_t* idx, int32_t n, int dir,
                  const ChainLayout& ch, cudaStream_t s) {
  (void)idx;
  if (n == 0)
    return 0;
  TmpBuf<int32_t> w(n, s), wmax(1, s);
  ell_width_kernel<<<grid_for(n), 256, 0, s>>>(ptr, n, dir, ch.chain_of.p, ch.cstart.p, w.p);
  count_launch();
  size_t bytes = 0;
  SFG_CUDA(cub::DeviceReduce::Max(nullptr, bytes, w.p, wmax.p, n, s));
  TmpBuf<char> tmp((int64_t)bytes, s);
  SFG_CUDA(cub::DeviceReduce::Max(tmp.p, bytes, w.p, wmax.p, n, s));
  int32_t h = 0;
  SFG_CUDA(cudaMemcpyAsync(&h, wmax.p, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  SFG_CUDA(cudaStreamSynchronize(s));
  return h;
}

void build_ell(const int32_t* ptr, const int32_t* idx, const double* val, int32_t n, int32_t S,
               int dir, int32_t CHN, const ChainLayout& ch, EllLayout& out, cudaStream_t s) {
  out.n = n;
  out.S = S;
  out.CHN = CHN;
  out.dir = dir;
  out.eidx.alloc((int64_t)(n > 0 ? n : 1) * CHN);
  out.eval.alloc((int64_t)(n > 0 ? n : 1) * (CHN + 2) * S);
  if (n == 0)
    return;
  ell_fill_kernel<<<grid_for(n), 256, 0, s>>>(ptr, idx, val, n, S, dir, CHN, ch.chain_of.p,
                                              ch.cstart.p, out.eidx.p, out.eval.p);
  count_launch();
  SFG_CUDA(cudaGetLastError());
  SFG_CUDA(cudaStreamSynchronize(s));
}

void launch_chain_ell(const EllArgs& a, int32_t CHN, cudaStream_t s) {
  if (a.seg_end <= a.seg_begin)
    return;
  switch (a.S) {
  case 2:
    launch_w<2>(a, CHN, s);
    break;
  case 4:
    launch_w<4>(a, CHN, s);
    break;
  case 8:
    launch_w<8>(a, CHN, s);
    break;
  case 16:
    launch_w<16>(a, CHN, s);
    break;
  case 32:
    launch_w<32>(a, CHN, s);
    break;
  default:
    throw InvalidArgument("chain-ELL executor needs 2..32 systems");
  }
}

} // namespace sfg
