// chainws.cu -- warp-specialised chain executor for batched solves (combos
// 1 and 8 with S >= 4 interleaved systems; see chain.cuh for the chains and
// ell.cuh for the fixed-width records it streams).
//
// A chain's tile period in the single-warp executors is the sum of the
// staging work for later tiles (row pointers -> indices -> value and x
// copies) and the tile's own dependent arithmetic, and on the critical path
// each chain level costs about one tile period.  Here every chain gets a
// PAIR of warps that share a ring of Q shared-memory slots:
//   loader warp  -- claims chains in chain-DAG level order, and for each tile
//                   copies the G chain-ELL records (values, carry coefficient,
//                   diagonal) with one bulk copy, the dependency indices with
//                   a second (prefetched a tile ahead), and gathers the x words
//                   of every dependency and the right-hand sides with per-lane
//                   cp.async; completion is counted on the slot's mbarrier;
//   compute warp -- waits for the slot, re-polls the words that were still
//                   unpublished when gathered, adds the terms in reference
//                   order, runs the carry through the G rows with shuffles,
//                   publishes, and releases the slot.
// so the compute warp's tile period is its arithmetic alone.
#include "common.cuh"
#include "ell.cuh"

namespace sfg {

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kMaxPairs = 8; // warp pairs per CTA (launch-time choice, 64 threads each)

__device__ __forceinline__ unsigned saddr(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mb_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(saddr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mb_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(saddr(bar)) : "memory");
}
__device__ __forceinline__ void mb_arrive_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(saddr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mb_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(saddr(bar)),
      "r"(parity)
      : "memory");
}
// arrive on `bar` once this thread's earlier cp.async copies have landed
__device__ __forceinline__ void cp_arrive_noinc(unsigned long long* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared.b64 [%0];" ::"r"(saddr(bar)) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
               "[%3];" ::"r"(saddr(dst)),
               "l"(src), "r"(bytes), "r"(saddr(bar))
               : "memory");
}
__device__ __forceinline__ void cp8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(saddr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

template <int S, int G, int CHN> struct alignas(16) WsSlot {
  double v[G][CHN + 2][S];         // G chain-ELL records: deps, carry coefficient, diagonal
  unsigned long long x[G][CHN][S]; // gathered dependency words
  unsigned long long rhs[G][S];
  int32_t idx[G][CHN];             // dependency rows (for re-polling)
  int32_t hdr[8];                  // end, bwd, p0, len, skew, tile
};

template <int S, int G, int CHN, int Q> struct alignas(16) WsPair {
  WsSlot<S, G, CHN> slot[Q];
  int32_t lidx[2][G][CHN]; // loader's index prefetch (tile t+1)
  unsigned long long full[Q], empty[Q], ibar[2];
};

template <int S, int G, int CHN, int Q>
__global__ void __launch_bounds__(kMaxPairs * 64) k_chain_ws(const EllArgs A) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  using Pair = WsPair<S, G, CHN, Q>;
  const int warp = threadIdx.x >> 5;
  Pair& W = reinterpret_cast<Pair*>(smem_raw)[warp >> 1];
  const bool loader = (warp & 1) == 0;
  const int lane = threadIdx.x & 31;
  const int k = lane / S;
  const int s = lane % S;
  constexpr unsigned kRec = (CHN + 2) * S * sizeof(double);
  constexpr unsigned kIdx = CHN * sizeof(int32_t);
  if (loader && lane == 0) {
    for (int q = 0; q < Q; ++q) {
      mb_init(&W.full[q], 33); // 32 cp.async arrivals + the bulk-copy arrival
      mb_init(&W.empty[q], 1);
    }
    mb_init(&W.ibar[0], 1);
    mb_init(&W.ibar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int n = A.n;
  const int total = A.seg_end - A.seg_begin;

  if (loader) {
    unsigned u = 0;  // slot uses
    unsigned lu = 0; // index-prefetch uses
    for (;;) {
      unsigned long long w0 = 0;
      if (lane == 0)
        w0 = atomicAdd(A.counter, 1ull);
      const long long wi = (long long)__shfl_sync(FULL, w0, 0);
      const int q = u % Q;
      if (u >= Q)
        mb_wait(&W.empty[q], ((u / Q) - 1) & 1);
      if (wi >= total) { // tell the compute warp to stop
        if (lane == 0)
          W.slot[q].hdr[0] = 1;
        __syncwarp();
        mb_arrive(&W.full[q]);
        if (lane == 0)
          mb_arrive(&W.full[q]);
        break;
      }
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
      const double* xo = bwd ? A.vout : A.vmid;
      const double* rv = bwd ? A.vmid : A.vin;
      auto issue_idx = [&](int t) { // indices of tile t -> lidx[lu & 1]
        const int q0 = p0 + G * t - skew;
        const int lo = max(q0, 0), hi = min(q0 + G, n);
        if (lane == 0) {
          unsigned long long* bar = &W.ibar[lu & 1];
          mb_arrive_tx(bar, (unsigned)(hi - lo) * kIdx);
          bulk_g2s(&W.lidx[lu & 1][lo - q0][0], eidx + (size_t)lo * CHN, (unsigned)(hi - lo) * kIdx,
                   bar);
        }
      };
      fence_proxy_async();
      __syncwarp();
      issue_idx(0);
      for (int t = 0; t < ntiles; ++t) {
        const int sl = u % Q;
        WsSlot<S, G, CHN>& SL = W.slot[sl];
        if (t > 0 && u >= Q) // (the first tile's slot was waited for above)
          mb_wait(&W.empty[sl], ((u / Q) - 1) & 1);
        const unsigned li = lu & 1;
        // prefetch the next tile's indices into the other buffer
        ++lu;
        if (t + 1 < ntiles) {
          fence_proxy_async();
          __syncwarp();
          issue_idx(t + 1);
        }
        const int q0 = p0 + G * t - skew;
        const int o = G * t - skew + k;
        const bool act = o >= 0 && o < len;
        const int pos = p0 + o;
        const int row = bwd ? n - 1 - pos : pos;
        mb_wait(&W.ibar[li], ((lu - 1) >> 1) & 1);
        if (lane == 0) {
          SL.hdr[0] = 0;
          SL.hdr[1] = bwd ? 1 : 0;
          SL.hdr[2] = p0;
          SL.hdr[3] = len;
          SL.hdr[4] = skew;
          SL.hdr[5] = t;
          SL.hdr[6] = item;
        }
        if (act) {
#pragma unroll
          for (int a = 0; a < CHN; ++a) {
            const int j = W.lidx[li][k][a];
            cp8(&SL.x[k][a][s], xo + (size_t)j * S + s);
          }
          for (int a = s; a < CHN; a += S)
            SL.idx[k][a] = W.lidx[li][k][a];
          cp8(&SL.rhs[k][s], rv + (size_t)row * S + s);
        }
        cp_arrive_noinc(&W.full[sl]);
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          const int lo = max(q0, 0), hi = min(q0 + G, n);
          mb_arrive_tx(&W.full[sl], (unsigned)(hi - lo) * kRec);
          bulk_g2s(&SL.v[lo - q0][0][0], eval + (size_t)lo * (CHN + 2) * S,
                   (unsigned)(hi - lo) * kRec, &W.full[sl]);
        }
        ++u;
      }
    }
    return;
  }

  // ---- compute warp
  unsigned u = 0;
  double carry = 0.0;
  for (;;) {
    const int sl = u % Q;
    WsSlot<S, G, CHN>& SL = W.slot[sl];
    mb_wait(&W.full[sl], (u / Q) & 1);
    if (SL.hdr[0])
      return;
    unsigned long long tr0 = 0, tr1 = 0;
    if (A.trace)
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr0));
    const bool bwd = SL.hdr[1] != 0;
    const int p0 = SL.hdr[2], len = SL.hdr[3], skew = SL.hdr[4], t = SL.hdr[5];
    if (t == 0)
      carry = 0.0;
    double* xo = bwd ? A.vout : A.vmid;
    const double* rv = bwd ? A.vmid : A.vin;
    const int kern = bwd ? 2 : 1;
    const int o = G * t - skew + k;
    const bool act = o >= 0 && o < len;
    const bool chained = o > 0;
    const int pos = p0 + o;
    const int row = bwd ? n - 1 - pos : pos;
    double acc = 0.0;
    const double d = act ? SL.v[k][CHN + 1][s] : 1.0;
    const double vc = act && chained ? SL.v[k][CHN][s] : 0.0;
    const double rd = __drcp_rn(d);
    if (act) {
      unsigned long long rw = SL.rhs[k][s];
      unsigned long long xx[CHN];
#pragma unroll
      for (int a = 0; a < CHN; ++a)
        xx[a] = SL.x[k][a][s];
      for (;;) {
        bool pending = is_sent_hi(rw);
#pragma unroll
        for (int a = 0; a < CHN; ++a)
          pending |= is_sent_hi(xx[a]);
        if (!pending)
          break;
        if (is_sent_hi(rw))
          rw = ld_relaxed_u64(rv + (size_t)row * S + s);
#pragma unroll
        for (int a = 0; a < CHN; ++a)
          if (is_sent_hi(xx[a]))
            xx[a] = ld_relaxed_u64(xo + (size_t)SL.idx[k][a] * S + s);
      }
      acc = __longlong_as_double((long long)rw);
#pragma unroll
      for (int a = 0; a < CHN; ++a)
        acc = __dsub_rn(acc, __dmul_rn(SL.v[k][a][s], __longlong_as_double((long long)xx[a])));
    }
    if (A.trace) {
      __syncwarp();
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr1));
    }
    if (act) {
      if (d == 0.0)
        report_error(A.err, kern, bwd ? n - 1 - row : row, row);
    }
    double x = 0.0;
#pragma unroll
    for (int kk = 0; kk < G; ++kk) {
      const double vv = chained ? __dsub_rn(acc, __dmul_rn(vc, carry)) : acc;
      const double q0 = __dmul_rn(vv, rd);
      double q = __fma_rn(__fma_rn(-q0, d, vv), rd, q0);
      const bool mine = act && k == kk;
      if (__builtin_expect(mine && !(exp_in_safe_range(vv) && exp_in_safe_range(d)), 0))
        q = ieee_div_slow(vv, d);
      if (mine) {
        x = q;
        publish_f64(xo + (size_t)row * S + s, q);
      }
      carry = __shfl_sync(FULL, x, kk * S + s);
    }
    if (A.ws_fence)
      __threadfence(); // drain this tile's published words to L2 before moving on
    __syncwarp();
    if (lane == 0) {
      mb_arrive(&W.empty[sl]);
      if (A.trace && t < A.trace_tiles) {
        unsigned long long te;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(te));
        unsigned long long* tr = A.trace + ((size_t)SL.hdr[6] * A.trace_tiles + t) * 3;
        tr[0] = tr0; // slot ready
        tr[1] = tr1; // dependencies ready and summed
        tr[2] = te;  // tile published
      }
    }
    ++u;
  }
}

template <int S, int G, int CHN, int Q> void launch_q(const EllArgs& a, cudaStream_t s) {
  auto kern = k_chain_ws<S, G, CHN, Q>;
  const int kPairs = a.ws_pairs >= 1 && a.ws_pairs <= kMaxPairs ? a.ws_pairs : 2;
  const size_t smem = (size_t)kPairs * sizeof(WsPair<S, G, CHN, Q>);
  SFG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  SFG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kPairs * 64, smem));
  if (per_sm < 1)
    per_sm = 1;
  if (a.blocks_per_sm > 0 && a.blocks_per_sm < per_sm)
    per_sm = a.blocks_per_sm;
  const int64_t items = a.seg_end - a.seg_begin;
  int64_t grid = (items + kPairs - 1) / kPairs;
  if (grid > (int64_t)per_sm * sm_count())
    grid = (int64_t)per_sm * sm_count();
  if (grid < 1)
    return;
  kern<<<(unsigned)grid, kPairs * 64, smem, s>>>(a);
  count_launch();
  SFG_CUDA(cudaGetLastError());
}

template <int S, int G, int CHN> void launch_c(const EllArgs& a, cudaStream_t s) {
  if (a.ws_slots <= 2)
    launch_q<S, G, CHN, 2>(a, s);
  else
    launch_q<S, G, CHN, 3>(a, s);
}

template <int S> void launch_s(const EllArgs& a, int32_t CHN, cudaStream_t s) {
  constexpr int G = 32 / S;
  if (CHN <= 4)
    launch_c<S, G, 4>(a, s);
  else if (CHN <= 8)
    launch_c<S, G, 8>(a, s);
  else if (CHN <= 12)
    launch_c<S, G, 12>(a, s);
  else
    launch_c<S, G, 16>(a, s);
}

} // namespace

void launch_chain_ws(const EllArgs& a, int32_t CHN, cudaStream_t s) {
  if (a.seg_end <= a.seg_begin)
    return;
  switch (a.S) {
  case 4:
    launch_s<4>(a, CHN, s);
    break;
  case 8:
    launch_s<8>(a, CHN, s);
    break;
  case 16:
    launch_s<16>(a, CHN, s);
    break;
  case 32:
    launch_s<32>(a, CHN, s);
    break;
  default:
    throw InvalidArgument("warp-specialised chain executor needs 4..32 systems");
  }
}

} // namespace sfg
