// chain.cu -- chain executor (see chain.cuh): inspector kernels that find
// the chains, their DAG levels, the warp batches and the SpMV tails, and the
// fused executor kernel.
#include "chain.cuh"
#include "common.cuh"


#ifndef SFG_CHAIN_MINB
#define SFG_CHAIN_MINB 1 // k_chain_sm blocks per SM it is compiled for (A/B builds)
#endif
#ifndef SFG_CHAIN_THREADS
// k_chain_sm block: one CTA of 12 warps per SM with up to 170 registers a
// thread measured fastest (C5 2.144 -> 1.942 ms against 2 CTAs of 8 warps at
// 128 registers; 8 warps 2.076, 10 warps 1.975, 13-16 warps 2.11-2.18 ms);
// the combo-1 staging buffers of 12 warps just fit in 227 KB
#define SFG_CHAIN_THREADS 384
#endif

#ifndef SFG_CHAIN_TRACE
// 1: the chain kernels record their tile timeline when SFG_TRACE is set
// (diagnostic builds: scripts/build_alt.sh trace "-DSFG_CHAIN_TRACE=1")
#define SFG_CHAIN_TRACE 0
#endif

#ifndef SFG_CHAIN_UNROLL
#define SFG_CHAIN_UNROLL 1 // unroll factor of k_chain_sm's tile loop (2: 2.42 ms, 3: 2.48 ms against 1.93 ms on C5)
#endif

#ifndef SFG_REFRESH
#define SFG_REFRESH 1 // re-stage a tile's dependency words before stage C (0: off, A/B builds)
#endif

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

namespace sfg {

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kThreads = 256;
constexpr int kSmThreads = SFG_CHAIN_THREADS;
constexpr int CH = 16; // dependencies staged in registers per batch

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

int bits_for(int64_t maxval) {
  int b = 1;
  while (b < 62 && (1ll << b) <= maxval)
    ++b;
  return b;
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ int pos_of(int j, int n, int dir) { return dir > 0 ? j : n - 1 - j; }

// ---------------------------------------------------------------------------
// inspector
// ---------------------------------------------------------------------------

// flag[p] = 1 if position p starts a chain: its last dependency is not p-1,
// or its second-to-last dependency is closer than G positions.
__global__ void chain_flag_kernel(const int32_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                                  int32_t n, int dir, int32_t G, int32_t* __restrict__ flag) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p <= n;
       p += (int64_t)gridDim.x * blockDim.x) {
    if (p == n) {
      flag[p] = 0;
      continue;
    }
    const int r = dir > 0 ? (int)p : n - 1 - (int)p;
    const int b = ptr[r], e = ptr[r + 1] - 1; // diagonal last
    const int cnt = e - b;
    bool chained = p > 0 && cnt >= 1 && pos_of(idx[e - 1], n, dir) == (int)p - 1;
    if (chained && cnt >= 2 && pos_of(idx[e - 2], n, dir) > (int)p - G)
      chained = false;
    flag[p] = chained ? 0 : 1;
  }
}

// split chains longer than max_len (flag pass 2)
__global__ void chain_cap_kernel(const int32_t* __restrict__ cid, const int32_t* __restrict__ cstart,
                                 int32_t n, int32_t max_len, int32_t* __restrict__ flag) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x)
    if (!flag[p] && ((int)p - cstart[cid[p]]) % max_len == 0)
      flag[p] = 1;
}

__global__ void chain_ids_kernel(const int32_t* __restrict__ flag, const int32_t* __restrict__ incl,
                                 int32_t n, int32_t* __restrict__ cid, int32_t* __restrict__ cstart) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p <= n;
       p += (int64_t)gridDim.x * blockDim.x) {
    if (p == n) {
      cstart[incl[n - 1]] = n;
      continue;
    }
    cid[p] = incl[p] - 1;
    if (flag[p])
      cstart[incl[p] - 1] = (int32_t)p;
  }
}

// chain level = 1 + max level of the chains its rows depend on (warp per
// chain, sync-free over ascending chain tickets).
__global__ void chain_levels_kernel(const int32_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                                    int32_t n, int dir, const int32_t* __restrict__ cstart,
                                    const int32_t* __restrict__ chain_of, int32_t nchain,
                                    int* level, unsigned long long* counter) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    unsigned long long c0 = 0;
    if (lane == 0)
      c0 = atomicAdd(counter, 1ull);
    const long long c = (long long)__shfl_sync(FULL, c0, 0);
    if (c >= nchain)
      break;
    const int p0 = __ldg(cstart + c), p1 = __ldg(cstart + c + 1);
    int lv = 1;
    for (int p = p0 + lane; p < p1; p += 32) {
      const int r = dir > 0 ? p : n - 1 - p;
      const int e = __ldg(ptr + r + 1) - 1;
      for (int q = __ldg(ptr + r); q < e; ++q) {
        const int pj = pos_of(__ldg(idx + q), n, dir);
        if (pj < p0) {
          const int l = poll_pos_i32(level + __ldg(chain_of + pj)) + 1;
          lv = l > lv ? l : lv;
        }
      }
    }
    lv = __reduce_max_sync(FULL, lv);
    if (lane == 0)
      st_relaxed_i32(level + c, lv);
  }
}

__global__ void iota_kernel(int32_t* a, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    a[i] = (int32_t)i;
}

__global__ void batch_flag_kernel(const int32_t* __restrict__ slev, int32_t nchain, int32_t CS,
                                  int32_t* __restrict__ rstart) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nchain;
       i += (int64_t)gridDim.x * blockDim.x)
    rstart[i] = (i == 0 || slev[i] != slev[i - 1]) ? (int32_t)i : 0;
}

__global__ void batch_flag2_kernel(const int32_t* __restrict__ rstart, int32_t nchain, int32_t CS,
                                   const int32_t* __restrict__ corder, int32_t* __restrict__ flag,
                                   int32_t* __restrict__ rank) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= nchain;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i == nchain) {
      flag[i] = 0;
      continue;
    }
    flag[i] = (((int32_t)i - rstart[i]) % CS == 0) ? 1 : 0;
    rank[corder[i]] = (int32_t)i;
  }
}

__global__ void batch_ptr_kernel(const int32_t* __restrict__ flag, const int32_t* __restrict__ bid,
                                 int32_t nchain, int32_t nbatch, int32_t* __restrict__ bptr) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= nchain;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i == nchain)
      bptr[nbatch] = nchain;
    else if (flag[i])
      bptr[bid[i]] = (int32_t)i;
  }
}

// SpMV row r -> the chain that comes last in claim order among those it reads
__global__ void tail_owner_kernel(const int32_t* __restrict__ ar_ptr,
                                  const int32_t* __restrict__ ar_idx,
                                  const int32_t* __restrict__ chain_of,
                                  const int32_t* __restrict__ rank,
                                  const int32_t* __restrict__ corder, int32_t n,
                                  int32_t* __restrict__ owner, int32_t* __restrict__ cnt) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    int best = -1, brank = -1;
    for (int p = ar_ptr[r]; p < ar_ptr[r + 1]; ++p) {
      const int c = chain_of[ar_idx[p]];
      if (rank[c] > brank) {
        brank = rank[c];
        best = c;
      }
    }
    if (best < 0)
      best = corder[0];
    owner[r] = best;
    atomicAdd(cnt + best, 1);
  }
}

__global__ void tail_scatter_kernel(const int32_t* __restrict__ owner, int32_t n,
                                    int32_t* __restrict__ cursor, int32_t* __restrict__ rows) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x)
    rows[atomicAdd(cursor + owner[r], 1)] = (int32_t)r;
}

// ---------------------------------------------------------------------------
// executor
// ---------------------------------------------------------------------------

// acc -= v_e * x[idx_e] for e in [b, eend), reference order; all loads of a
// batch of CH entries are issued before the first one is consumed.
template <int S>
__device__ __noinline__ double partial_sum(double acc, int b, int eend,
                                              const int32_t* __restrict__ idx,
                                              const double* __restrict__ val, const double* x,
                                              int s) {
  for (int p = b; p < eend; p += CH) {
    const int cnt = min(CH, eend - p);
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
        const double xj = xx[a] != SENT ? __longlong_as_double((long long)xx[a])
                                        : poll_f64(x + (size_t)jj[a] * S + s, 0);
        acc = __dsub_rn(acc, __dmul_rn(vv[a], xj));
      }
  }
  return acc;
}

// One row of a tile as staged by the software pipeline: its non-carry
// dependencies (indices, values, a first speculative read of each x word),
// diagonal, carry coefficient, RN(1/diagonal) and right-hand side.
template <int CHN> struct Stage {
  int r, b, eend;
  bool act, chained;
  int jj[CHN];
  double vv[CHN];
  unsigned long long xx[CHN];
  double d, vc, rd;
  unsigned long long rhs;
};

// Waits until every staged x word of the row is published (all still-SENT
// words are re-read together each round), then adds all terms in the
// reference order with straight-line code.  Full-width rows (the common
// case) take a path without per-term predicates.
template <int S, int CHN>
__device__ __forceinline__ double wait_and_sum(Stage<CHN>& st, double acc,
                                               const int32_t* __restrict__ idx,
                                               const double* __restrict__ val, const double* xv) {
  const int cnt = st.eend - st.b;
  if (cnt == CHN) {
    for (;;) {
      bool pending = false;
#pragma unroll
      for (int a = 0; a < CHN; ++a)
        pending |= is_sent_hi(st.xx[a]);
      if (!pending)
        break;
#pragma unroll
      for (int a = 0; a < CHN; ++a)
        if (is_sent_hi(st.xx[a]))
          st.xx[a] = ld_relaxed_u64(xv + (size_t)st.jj[a] * S);
    }
#pragma unroll
    for (int a = 0; a < CHN; ++a)
      acc = __dsub_rn(acc, __dmul_rn(st.vv[a], __longlong_as_double((long long)st.xx[a])));
    return acc;
  }
  const int m = cnt < CHN ? cnt : CHN;
  for (;;) {
    bool pending = false;
#pragma unroll
    for (int a = 0; a < CHN; ++a)
      pending |= a < m && is_sent_hi(st.xx[a]);
    if (!pending)
      break;
#pragma unroll
    for (int a = 0; a < CHN; ++a)
      if (a < m && is_sent_hi(st.xx[a]))
        st.xx[a] = ld_relaxed_u64(xv + (size_t)st.jj[a] * S);
  }
#pragma unroll
  for (int a = 0; a < CHN; ++a)
    if (a < m)
      acc = __dsub_rn(acc, __dmul_rn(st.vv[a], __longlong_as_double((long long)st.xx[a])));
  for (int p = st.b + CHN; p < st.eend; ++p) // rows longer than the staging width
    acc = __dsub_rn(acc, __dmul_rn(__ldg(val + (size_t)p * S),
                                   poll_f64(xv + (size_t)__ldg(idx + p) * S, 0)));
  return acc;
}

// One warp per chain.  Lane = (row-in-tile k, system s), G = 32/S rows in
// flight (<= 8).  Tiles are skewed by the chain level (offset = level mod G)
// so that tile t of a chain needs at most tile t of the chains of the
// previous level.  A four-stage software pipeline keeps every load off the
// critical path: iteration t issues the row-pointer loads of tile t+3, the
// dependency-index loads of tile t+2 and the value / x loads of tile t+1 --
// none of which waits on a load issued in the same iteration -- and then
// completes tile t: all rows pre-add their already-available terms in
// parallel, then row k, at its turn, adds the rest, applies the carry
// x_{p-1} received by shuffle, divides with the staged reciprocal and
// publishes.
template <int S, int G, int CHN, int COMBO>
__global__ void __launch_bounds__(kThreads) k_chain(const ChainArgs A) {
  const int lane = threadIdx.x & 31;
  const int k = lane / S;
  const int s = lane % S;
  const bool lane_on = k < G;
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
    const int32_t* ptr = bwd ? A.lt_ptr : A.lr_ptr;
    const int32_t* idx = bwd ? A.lt_idx : A.lr_idx;
    const double* val = bwd ? A.lt_val : A.lr_val;
    const int32_t* cstart = bwd ? A.b_cstart : A.f_cstart;
    const int32_t* corder = bwd ? A.b_corder : A.f_corder;
    const int32_t* bptr = bwd ? A.b_bptr : A.f_bptr;
    const int32_t* clev = bwd ? A.b_level : A.f_level;
    const int c = __ldg(corder + __ldg(bptr + bi));
    const int p0 = __ldg(cstart + c);
    const int len = __ldg(cstart + c + 1) - p0;
    const int skew = (__ldg(clev + c) * A.skew_mul) % G;
    const int ntiles = (len + skew + G - 1) / G;
    double* xo = bwd ? A.vout : A.vmid;
    const double* rhs_vec = bwd ? A.vmid : A.vin;
    const int kern = bwd ? 2 : 1;
    const bool pass1 = COMBO != 1 || (A.phase & 1);
    const bool pass2 = COMBO == 1 && (A.phase & 2);
    const bool solve = COMBO != 4 || (A.phase & 1);
    // vectors the staged x words / right-hand sides come from
    const double* xs = pass1 ? xo : A.vout;
    const double* rs = pass1 ? rhs_vec : A.vmid;
    const bool rpoll = pass1 ? bwd : true;
    unsigned long long* tr =
        SFG_CHAIN_TRACE && A.trace ? A.trace + (size_t)item * A.trace_tiles * 3 : nullptr;
    const unsigned long long t_claim = tr ? gtimer() : 0ull;
    if (solve) {
      auto row_of = [&](int o) { const int p = p0 + o; return bwd ? A.n - 1 - p : p; };
      auto active = [&](int tile) {
        const int o = G * tile - skew + k;
        return lane_on && tile >= 0 && tile < ntiles && o >= 0 && o < len;
      };
      // pipeline registers
      int pb3 = 0, pe3 = 0;          // tile t+3: ptr[r], ptr[r+1]
      int b2 = 0, eend2 = 0, e2 = 0; // tile t+2: geometry
      bool act2 = false;
      int idx2[CHN];                 // tile t+2: dependency indices
      Stage<CHN> cur;                // tile t (loaded during iteration t-1)
      cur.act = false;
      cur.b = cur.eend = 0;
      double carry = 0.0, carry2 = 0.0;
#pragma unroll 1
      for (int t = -3; t < ntiles; ++t) {
        // stage A: row pointers of tile t+3
        const bool act3 = active(t + 3);
        int npb = 0, npe = 0;
        if (act3) {
          const int r = row_of(G * (t + 3) - skew + k);
          npb = __ldg(ptr + r);
          npe = __ldg(ptr + r + 1);
        }
        // stage B: dependency indices of tile t+2 (pointers from stage A of t-1)
        const bool nact2 = active(t + 2);
        int nb2 = 0, ne2 = 0, neend2 = 0;
        int nidx2[CHN];
        if (nact2) {
          nb2 = pb3;
          ne2 = pe3 - 1;
          neend2 = (G * (t + 2) - skew + k) > 0 ? ne2 - 1 : ne2;
          const int32_t* ib = idx + nb2;
          if (neend2 - nb2 >= CHN) {
#pragma unroll
            for (int a = 0; a < CHN; ++a)
              nidx2[a] = __ldg(ib + a);
          } else {
#pragma unroll
            for (int a = 0; a < CHN; ++a)
              if (a < neend2 - nb2)
                nidx2[a] = __ldg(ib + a);
          }
        }
        // stage C: values and first x reads of tile t+1 (indices from stage B of t-1)
        Stage<CHN> nxt;
        nxt.act = act2;
        nxt.b = 0;
        nxt.eend = 0;
        if (act2) {
          const int o = G * (t + 1) - skew + k;
          nxt.chained = o > 0;
          nxt.r = row_of(o);
          nxt.b = b2;
          nxt.eend = eend2;
          nxt.d = __ldg(val + (size_t)e2 * S + s);
          nxt.vc = nxt.chained ? __ldg(val + (size_t)(e2 - 1) * S + s) : 0.0;
          nxt.rhs = rpoll ? ld_relaxed_u64(rs + (size_t)nxt.r * S + s)
                          : (unsigned long long)__double_as_longlong(
                                __ldg(rs + (size_t)nxt.r * S + s));
          const int cnt = eend2 - b2;
          const double* vb = val + (size_t)b2 * S + s;
          const double* xb = xs + s;
          if (cnt >= CHN) {
#pragma unroll
            for (int a = 0; a < CHN; ++a) {
              nxt.jj[a] = idx2[a];
              nxt.vv[a] = __ldg(vb + a * S);
              nxt.xx[a] = ld_relaxed_u64(xb + (size_t)idx2[a] * S);
            }
          } else {
#pragma unroll
            for (int a = 0; a < CHN; ++a)
              if (a < cnt) {
                nxt.jj[a] = idx2[a];
                nxt.vv[a] = __ldg(vb + a * S);
                nxt.xx[a] = ld_relaxed_u64(xb + (size_t)idx2[a] * S);
              }
          }
        }
        // stage D: complete tile t
        if (t >= 0) {
          const unsigned long long t_part = tr ? gtimer() : 0ull;
          const int r = cur.r;
          double x = 0.0;
          if (pass1) {
            // wait phase: every row of the tile gathers its non-carry terms
            double acc = 0.0;
            if (cur.act) {
              // only a published right-hand side (vmid) is polled: b is read
              // once, and may hold any bit pattern
              const double rv = (!rpoll || cur.rhs != SENT)
                                    ? __longlong_as_double((long long)cur.rhs)
                                    : poll_f64(rhs_vec + (size_t)r * S + s, 0);
              acc = wait_and_sum<S, CHN>(cur, rv, idx, val + s, xo + s);
              if (cur.d == 0.0)
                report_error(A.err, kern, bwd ? A.n - 1 - r : r, r);
            }
            // carry phase: every lane evaluates its row with the broadcast
            // carry, group kk keeps and publishes it (no divergent region)
#pragma unroll
            for (int kk = 0; kk < G; ++kk) {
              const double v = cur.chained ? __dsub_rn(acc, __dmul_rn(cur.vc, carry)) : acc;
              const double q0 = __dmul_rn(v, cur.rd);
              double q = __fma_rn(__fma_rn(-q0, cur.d, v), cur.rd, q0);
              const bool mine = cur.act && k == kk;
              if (__builtin_expect(mine && !(exp_in_safe_range(v) && exp_in_safe_range(cur.d)), 0))
                q = ieee_div_slow(v, cur.d);
              if (mine) {
                x = q;
                publish_f64(xo + (size_t)r * S + s, q);
              }
              carry = __shfl_sync(FULL, x, kk * S + s);
            }
          }
          if (pass2) { // combo 1: x2 = inv(L) z on the same rows
            double x2 = 0.0;
#pragma unroll 1
            for (int kk = 0; kk < G; ++kk) {
              if (cur.act && k == kk) {
                const double z =
                    pass1 ? x
                          : (cur.rhs != SENT ? __longlong_as_double((long long)cur.rhs)
                                             : poll_f64(A.vmid + (size_t)r * S + s, 0));
                const double acc2 = pass1
                                        ? partial_sum<S>(z, cur.b, cur.eend, idx, val, A.vout, s)
                                        : wait_and_sum<S, CHN>(cur, z, idx, val + s, A.vout + s);
                if (cur.d == 0.0)
                  report_error(A.err, 2, r, r);
                x2 = cur.chained ? div_with_rcp(__dsub_rn(acc2, __dmul_rn(cur.vc, carry2)), cur.d,
                                                cur.rd)
                                 : div_with_rcp(acc2, cur.d, cur.rd);
                publish_f64(A.vout + (size_t)r * S + s, x2);
              }
              carry2 = __shfl_sync(FULL, x2, kk * S + s);
            }
          }
          if (tr && lane == 0 && t < A.trace_tiles) {
            tr[t * 3 + 0] = t_claim;
            tr[t * 3 + 1] = t_part;
            tr[t * 3 + 2] = gtimer();
          }
        }
        // rotate the pipeline; the reciprocal of the next tile's diagonal
        // is computed here, long before its carry pass needs it
        if (nxt.act)
          nxt.rd = __drcp_rn(nxt.d);
        cur = nxt;
        act2 = nact2;
        b2 = nb2;
        e2 = ne2;
        eend2 = neend2;
#pragma unroll
        for (int a = 0; a < CHN; ++a)
          idx2[a] = nidx2[a];
        pb3 = npb;
        pe3 = npe;
      }
    }
    if (COMBO == 4 && (A.phase & 2)) {
      // SpMV rows whose last input chain is this warp's chain: the row
      // gather adds terms in the sequential CSC scatter's order
      for (int tq = __ldg(A.tail_ptr + c) + lane; tq < __ldg(A.tail_ptr + c + 1); tq += 32) {
        const int yr = __ldg(A.tail_rows + tq);
        double acc = 0.0;
        for (int p = __ldg(A.ar_ptr + yr); p < __ldg(A.ar_ptr + yr + 1); ++p)
          acc = __dadd_rn(acc, __dmul_rn(__ldg(A.ar_val + p),
                                         poll_f64(A.vmid + __ldg(A.ar_idx + p), 0)));
        A.vout[yr] = acc;
      }
    }
  }
}


// ---------------------------------------------------------------------------
// Shared-memory-staged variant for S >= 2 systems (the batched solves).
// Stage C copies the next tile's values and first x reads into a per-warp
// double buffer with cp.async.cg (16-byte, L2-coherent: the pair of systems
// s, s+1 of one nonzero / one x row is contiguous), so the staged data holds
// no registers while in flight and twice as many warps fit on an SM.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cp_async_cg16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait1() {
  asm volatile("cp.async.wait_group 1;" ::: "memory");
}

// X2 (fused combo 1): the second solve's words x2[idx] are staged with the
// first's, so both passes of a tile share the staged values of L.
template <int S, int G, int CHN, bool X2 = false> struct StageBuf {
  double v[G][CHN][S];
  unsigned long long x[G][CHN][S];
  unsigned long long x2[X2 ? G : 1][X2 ? CHN : 1][S];
};

template <int S, int G, int CHN, int COMBO>
__global__ void __launch_bounds__(kSmThreads, COMBO == 1 ? 1 : SFG_CHAIN_MINB) k_chain_sm(const ChainArgs A) {
  static_assert(S >= 2 && S % 2 == 0, "pair copies need an even number of systems");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr bool X2 = COMBO == 1;
  using Buf = StageBuf<S, G, CHN, X2>;
  Buf* wbuf = reinterpret_cast<Buf*>(smem_raw) + 2 * (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const int k = lane / S;
  const int s = lane % S;
  const bool lane_on = k < G;
  const bool copier = (s & 1) == 0;
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
    const int32_t* ptr = bwd ? A.lt_ptr : A.lr_ptr;
    const int32_t* idx = bwd ? A.lt_idx : A.lr_idx;
    const double* val = bwd ? A.lt_val : A.lr_val;
    const int32_t* cstart = bwd ? A.b_cstart : A.f_cstart;
    const int32_t* corder = bwd ? A.b_corder : A.f_corder;
    const int32_t* bptr = bwd ? A.b_bptr : A.f_bptr;
    const int32_t* clev = bwd ? A.b_level : A.f_level;
    const int c = __ldg(corder + __ldg(bptr + bi));
    const int p0 = __ldg(cstart + c);
    const int len = __ldg(cstart + c + 1) - p0;
    const int skew = (__ldg(clev + c) * A.skew_mul) % G;
    const int ntiles = (len + skew + G - 1) / G;
    double* xo = bwd ? A.vout : A.vmid;
    const double* rhs_vec = bwd ? A.vmid : A.vin;
    const int kern = bwd ? 2 : 1;
    const bool pass1 = COMBO != 1 || (A.phase & 1);
    const bool pass2 = COMBO == 1 && (A.phase & 2);
    const double* xs = pass1 ? xo : A.vout;
    const double* rs = pass1 ? rhs_vec : A.vmid;
    const bool rpoll = pass1 ? bwd : true;
    unsigned long long* tr =
        SFG_CHAIN_TRACE && A.trace ? A.trace + (size_t)item * A.trace_tiles * 3 : nullptr;
    const unsigned long long t_claim = tr ? gtimer() : 0ull;
    auto row_of = [&](int o) { const int p = p0 + o; return bwd ? A.n - 1 - p : p; };
    auto active = [&](int tile) {
      const int o = G * tile - skew + k;
      return lane_on && tile >= 0 && tile < ntiles && o >= 0 && o < len;
    };
    int pb3 = 0, pe3 = 0;
    int b2 = 0, eend2 = 0, e2 = 0;
    bool act2 = false;
    int idx2[CHN];
    // current tile (scalars in registers, values / x words in smem)
    int cr = 0, cb = 0, ceend = 0;
    bool cact = false, cchained = false;
    int cjj[CHN];
    double cd = 1.0, cvc = 0.0, crd = 1.0;
    unsigned long long crhs = 0;
    double carry = 0.0, carry2 = 0.0;
    if (COMBO == 8 && (A.phase & 1) && A.bwd_reset) {
      // Fused fwd -> bwd: the backward outputs are reset here, not by k_prep
      // before the launch.  The last bwd_reset_items forward work items --
      // the top levels, claimed long before their producers finish, so their
      // warps would otherwise only wait -- each set one slice of vout to
      // SENT first; every backward chain waits for all slices before it
      // reads a vout word.  (The unfused pair resets vout between its two
      // launches.)
      const int ri = A.f_nbatch - 1 - item;
      if (!bwd && ri < A.bwd_reset_items) {
        const int64_t w2 = A.bwd_reset_words / 2; // 16-byte stores
        const int64_t per = (w2 + A.bwd_reset_items - 1) / A.bwd_reset_items;
        const int64_t lo = per * ri, hi = min(w2, lo + per);
        ulonglong2* p2 = reinterpret_cast<ulonglong2*>(A.bwd_reset);
        for (int64_t i = lo + lane; i < hi; i += 32)
          p2[i] = make_ulonglong2(SENT, SENT);
        __syncwarp();
        if (lane == 0) {
          __threadfence();
          atomicAdd(A.reset_done, 1ull);
        }
      }
      if (bwd) {
        if (lane == 0)
          while (ld_relaxed_u64(A.reset_done) < (unsigned long long)A.bwd_reset_items)
            __nanosleep(200);
        __threadfence();
      }
    }
    if (bwd && pass1 && (A.phase & 1) && A.bwd_gate) { // fused launch only
      // a backward chain cannot start before the forward solve has reached
      // its first right-hand side: one lane sleeps on that word instead of
      // the whole warp polling L2 while the forward solve still runs
      if (lane == 0) {
        const unsigned long long* w = reinterpret_cast<const unsigned long long*>(
            rhs_vec + (size_t)row_of(0) * S);
        while (is_sent_hi(ld_relaxed_u64(w)))
          __nanosleep(A.bwd_gate);
      }
    }
    __syncwarp();
#if SFG_CHAIN_UNROLL > 1
    constexpr int kUnrollT = SFG_CHAIN_UNROLL;
#pragma unroll kUnrollT
#else
#pragma unroll 1
#endif
    for (int t = -3; t < ntiles; ++t) {
      // stage A: row pointers of tile t+3
      int npb = 0, npe = 0;
      if (active(t + 3)) {
        const int r = row_of(G * (t + 3) - skew + k);
        npb = __ldg(ptr + r);
        npe = __ldg(ptr + r + 1);
      }
      // stage B: dependency indices of tile t+2
      const bool nact2 = active(t + 2);
      int nb2 = 0, ne2 = 0, neend2 = 0;
      int nidx2[CHN];
      if (nact2) {
        nb2 = pb3;
        ne2 = pe3 - 1;
        neend2 = (G * (t + 2) - skew + k) > 0 ? ne2 - 1 : ne2;
        const int32_t* ib = idx + nb2;
        const int m = neend2 - nb2;
#pragma unroll
        for (int a = 0; a < CHN; ++a)
          if (a < m)
            nidx2[a] = __ldg(ib + a);
        // the row's values (entries nb2 .. ne2, S doubles each) HBM -> L2
        // now, so stage C's copies of them one iteration later hit L2
        const int lines = ((ne2 - nb2 + 1) * S * 8 + 127) >> 7;
        if (s < lines)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(val + (size_t)nb2 * S + s * 16));
      }
#if SFG_REFRESH
      // re-copy the dependency words of tile t (staged one iteration ago)
      // now, so stage D checks a snapshot taken one stage C earlier rather
      // than a whole iteration earlier: words published in between need no
      // re-poll round trip (C5 2.167 -> 2.144 ms kernel; the same copy at the
      // top of the iteration 2.153 ms).  Either copy may land last; both read
      // a word that is written once, so the slot holds the sentinel or the
      // value.
      if (t >= 0 && cact && copier) {
        const int m = ceend - cb < CHN ? ceend - cb : CHN;
        Buf& rb = wbuf[t & 1];
#pragma unroll
        for (int a = 0; a < CHN; ++a)
          if (a < m)
            cp_async_cg16(&rb.x[k][a][s], xs + s + (size_t)cjj[a] * S);
      }
      cp_async_commit();
#endif
      // stage C: tile t+1 -> smem buffer (t+1)&1 by 16-byte async copies
      Buf& nb = wbuf[(t + 1) & 1];
      int nr = 0;
      bool nchained = false;
      double nd = 1.0, nvc = 0.0;
      unsigned long long nrhs = 0;
      if (act2) {
        const int o = G * (t + 1) - skew + k;
        nchained = o > 0;
        nr = row_of(o);
        nd = __ldg(val + (size_t)e2 * S + s);
        nvc = nchained ? __ldg(val + (size_t)(e2 - 1) * S + s) : 0.0;
        nrhs = rpoll ? ld_relaxed_u64(rs + (size_t)nr * S + s)
                     : (unsigned long long)__double_as_longlong(__ldg(rs + (size_t)nr * S + s));
        if (copier) {
          const int m = eend2 - b2;
          const double* vb = val + (size_t)b2 * S + s;
          const double* xb = xs + s;
#pragma unroll
          for (int a = 0; a < CHN; ++a)
            if (a < m) {
              cp_async_cg16(&nb.v[k][a][s], vb + a * S);
              // combo 1 leaves these words to the refresh copy one stage
              // before stage D (fwd->fwd 1.473 -> 1.408 ms; combo 8 measured
              // 1.940 -> 2.021 ms without its early copy)
              if (!(SFG_REFRESH && X2))
                cp_async_cg16(&nb.x[k][a][s], xb + (size_t)idx2[a] * S);
              if (X2 && pass1 && pass2)
                cp_async_cg16(&nb.x2[X2 ? k : 0][X2 ? a : 0][s], A.vout + s + (size_t)idx2[a] * S);
            }
        }
      }
      cp_async_commit();
      // stage D: complete tile t from smem buffer t&1
      if (t >= 0) {
        const long long c0 = tr ? clock64() : 0;
        cp_async_wait1();
        __syncwarp();
        const unsigned long long t_part = tr ? gtimer() : 0ull;
        long long c1 = 0;
        unsigned long long t_ready = 0;
        const Buf& cbuf = wbuf[t & 1];
        const int r = cr;
        double x = 0.0;
        if (pass1) {
          double acc = 0.0;
          if (cact) {
            // only a published right-hand side (vmid) is polled: b is read
            // once, and may hold any bit pattern
            acc = (!rpoll || crhs != SENT) ? __longlong_as_double((long long)crhs)
                                           : poll_f64(rhs_vec + (size_t)r * S + s, 0);
            const int m = ceend - cb < CHN ? ceend - cb : CHN;
            unsigned long long xx[CHN];
#pragma unroll
            for (int a = 0; a < CHN; ++a)
              if (a < m)
                xx[a] = cbuf.x[k][a][s];
            for (;;) {
              bool pending = false;
#pragma unroll
              for (int a = 0; a < CHN; ++a)
                pending |= a < m && is_sent_hi(xx[a]);
              if (!pending)
                break;
#pragma unroll
              for (int a = 0; a < CHN; ++a)
                if (a < m && is_sent_hi(xx[a]))
                  xx[a] = ld_relaxed_u64(xo + (size_t)cjj[a] * S + s);
            }
#pragma unroll
            for (int a = 0; a < CHN; ++a)
              if (a < m)
                acc = __dsub_rn(acc, __dmul_rn(cbuf.v[k][a][s],
                                               __longlong_as_double((long long)xx[a])));
            for (int p = cb + CHN; p < ceend; ++p) // rows longer than the staging width
              acc = __dsub_rn(acc, __dmul_rn(__ldg(val + (size_t)p * S + s),
                                             poll_f64(xo + (size_t)__ldg(idx + p) * S + s, 0)));
            if (cd == 0.0)
              report_error(A.err, kern, bwd ? A.n - 1 - r : r, r);
          }
          if (tr) {
            c1 = clock64();
            t_ready = gtimer();
          }
#pragma unroll
          for (int kk = 0; kk < G; ++kk) {
            const double v = cchained ? __dsub_rn(acc, __dmul_rn(cvc, carry)) : acc;
            const double q0 = __dmul_rn(v, crd);
            double q = __fma_rn(__fma_rn(-q0, cd, v), crd, q0);
            const bool mine = cact && k == kk;
            if (__builtin_expect(mine && !(exp_in_safe_range(v) && exp_in_safe_range(cd)), 0))
              q = ieee_div_slow(v, cd);
            if (mine) {
              x = q;
              publish_f64(xo + (size_t)r * S + s, q);
            }
            carry = __shfl_sync(FULL, x, kk * S + s);
          }
        }
        if (pass2) { // combo 1: x2 = inv(L) z on the same rows
          double acc2 = 0.0;
          if (cact) {
            const double z = pass1 ? x
                                   : (crhs != SENT ? __longlong_as_double((long long)crhs)
                                                   : poll_f64(A.vmid + (size_t)r * S + s, 0));
            // the words were staged with the tile (x2 beside x when fused,
            // in x when the second solve runs alone)
            const int m = ceend - cb < CHN ? ceend - cb : CHN;
            unsigned long long xx[CHN];
#pragma unroll
            for (int a = 0; a < CHN; ++a)
              if (a < m)
                xx[a] = (X2 && pass1) ? cbuf.x2[X2 ? k : 0][X2 ? a : 0][s] : cbuf.x[k][a][s];
            for (;;) {
              bool pending = false;
#pragma unroll
              for (int a = 0; a < CHN; ++a)
                pending |= a < m && is_sent_hi(xx[a]);
              if (!pending)
                break;
#pragma unroll
              for (int a = 0; a < CHN; ++a)
                if (a < m && is_sent_hi(xx[a]))
                  xx[a] = ld_relaxed_u64(A.vout + (size_t)cjj[a] * S + s);
            }
            acc2 = z;
#pragma unroll
            for (int a = 0; a < CHN; ++a)
              if (a < m)
                acc2 = __dsub_rn(acc2, __dmul_rn(cbuf.v[k][a][s],
                                                 __longlong_as_double((long long)xx[a])));
            for (int p = cb + CHN; p < ceend; ++p) // rows longer than the staging width
              acc2 = __dsub_rn(acc2, __dmul_rn(__ldg(val + (size_t)p * S + s),
                                               poll_f64(A.vout + (size_t)__ldg(idx + p) * S + s, 0)));
            if (cd == 0.0)
              report_error(A.err, 2, r, r);
          }
          double x2 = 0.0;
#pragma unroll
          for (int kk = 0; kk < G; ++kk) {
            const double v = cchained ? __dsub_rn(acc2, __dmul_rn(cvc, carry2)) : acc2;
            const double q0 = __dmul_rn(v, crd);
            double q = __fma_rn(__fma_rn(-q0, cd, v), crd, q0);
            const bool mine = cact && k == kk;
            if (__builtin_expect(mine && !(exp_in_safe_range(v) && exp_in_safe_range(cd)), 0))
              q = ieee_div_slow(v, cd);
            if (mine) {
              x2 = q;
              publish_f64(A.vout + (size_t)r * S + s, q);
            }
            carry2 = __shfl_sync(FULL, x2, kk * S + s);
          }
        }
        if (tr && lane == 0 && t < A.trace_tiles) {
          // {stage-D entry after the copy wait (globaltimer ns),
          //  chain id << 44 | ns from entry to every term summed << 22 | carry
          //  cycles, tile end (globaltimer ns)}
          const long long c2 = clock64();
          const unsigned long long lim = (1ull << 22) - 1;
          const unsigned long long dr = pass1 ? t_ready - t_part : 0ull;
          const unsigned long long cc = (unsigned long long)(c2 - c1);
          tr[t * 3 + 0] = t_part;
          tr[t * 3 + 1] = ((unsigned long long)c << 44) | ((dr < lim ? dr : lim) << 22) | (cc < lim ? cc : lim);
          tr[t * 3 + 2] = gtimer();
          (void)t_claim;
          (void)c0;
        }
      }
      // rotate
      cr = nr;
      cb = b2;
      ceend = eend2;
      cact = act2;
      cchained = nchained;
      cd = nd;
      cvc = nvc;
      crd = act2 ? __drcp_rn(nd) : 1.0;
      crhs = nrhs;
#pragma unroll
      for (int a = 0; a < CHN; ++a)
        cjj[a] = idx2[a];
      act2 = nact2;
      b2 = nb2;
      e2 = ne2;
      eend2 = neend2;
#pragma unroll
      for (int a = 0; a < CHN; ++a)
        idx2[a] = nidx2[a];
      pb3 = npb;
      pe3 = npe;
    }
    // drain this warp's async copies before its buffers are reused
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncwarp();
  }
}

template <int S, int G, int COMBO> void launch_g(const ChainArgs& a, cudaStream_t s) {
  constexpr int CHN = 12;
  constexpr bool use_sm = S >= 2 && S % 2 == 0 && COMBO != 4;
  auto kern = use_sm ? k_chain_sm<(S >= 2 ? S : 2), G, CHN, COMBO> : k_chain<S, G, CHN, COMBO>;
  const size_t smem =
      use_sm ? (size_t)(kSmThreads / 32) * 2 * sizeof(StageBuf<(S >= 2 ? S : 2), G, CHN, COMBO == 1>) : 0;
  if (smem > 48 * 1024)
    SFG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  SFG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, use_sm ? kSmThreads : kThreads, smem));
  if (per_sm < 1)
    per_sm = 1;
  if (a.blocks_per_sm > 0 && a.blocks_per_sm < per_sm)
    per_sm = a.blocks_per_sm;
  const int64_t items = a.seg_end - a.seg_begin;
  const int threads = use_sm ? kSmThreads : kThreads;
  int64_t grid = (items + (threads / 32) - 1) / (threads / 32);
  if (grid > (int64_t)per_sm * sm_count())
    grid = (int64_t)per_sm * sm_count();
  if (grid < 1)
    return;
  kern<<<(unsigned)grid, threads, smem, s>>>(a);
  count_launch();
  SFG_CUDA(cudaGetLastError());
}

// Tile height G (rows in flight per chain): chain_G (chain.cuh); a.tile_rows
// (a power of two with G * S <= 32) overrides it.
template <int S, int COMBO> void launch_t(const ChainArgs& a, cudaStream_t s) {
  constexpr int G = S <= 8 ? 4 : 32 / S; // chain_G's default (chain.cuh)
  if (a.tile_rows > 0 && a.tile_rows != G && a.tile_rows * S <= 32) {
    switch (a.tile_rows) {
    case 1:
      launch_g<S, 1, COMBO>(a, s);
      return;
    case 2:
      if constexpr (2 * S <= 32)
        launch_g<S, 2, COMBO>(a, s);
      return;
    case 4:
      if constexpr (4 * S <= 32)
        launch_g<S, 4, COMBO>(a, s);
      return;
    case 8:
      if constexpr (8 * S <= 32)
        launch_g<S, 8, COMBO>(a, s);
      return;
    case 16:
      if constexpr (16 * S <= 32 && S >= 2)
        launch_g<S, 16, COMBO>(a, s);
      return;
    default:
      break;
    }
  }
  launch_g<S, G, COMBO>(a, s);
}

template <int COMBO> void launch_c(const ChainArgs& a, cudaStream_t s) {
  switch (a.S) {
  case 1:
    launch_t<1, COMBO>(a, s);
    break;
  case 2:
    launch_t<2, COMBO>(a, s);
    break;
  case 4:
    launch_t<4, COMBO>(a, s);
    break;
  case 8:
    launch_t<8, COMBO>(a, s);
    break;
  case 16:
    launch_t<16, COMBO>(a, s);
    break;
  case 32:
    launch_t<32, COMBO>(a, s);
    break;
  default:
    throw InvalidArgument("nsys must be a power of two <= 32");
  }
}

} // namespace

void build_chains(const int32_t* ptr, const int32_t* idx, int32_t n, int dir, int32_t G,
                  int32_t CS, int32_t max_len, ChainLayout& out, cudaStream_t s) {
  out.n = n;
  out.G = G;
  out.CS = CS;
  out.dir = dir;
  if (n == 0) {
    out.nchain = out.nbatch = 0;
    out.cstart.alloc(1);
    out.batch_ptr.alloc(1);
    out.corder.alloc(1);
    out.chain_of.alloc(1);
    out.rank.alloc(1);
    SFG_CUDA(cudaMemsetAsync(out.cstart.p, 0, sizeof(int32_t), s));
    SFG_CUDA(cudaMemsetAsync(out.batch_ptr.p, 0, sizeof(int32_t), s));
    return;
  }
  TmpBuf<int32_t> flag((int64_t)n + 1, s), incl((int64_t)n + 1, s);
  out.chain_of.alloc(n);
  chain_flag_kernel<<<grid_for((int64_t)n + 1), 256, 0, s>>>(ptr, idx, n, dir, G, flag.p);
  count_launch();
  size_t bytes = 0;
  auto scan_ids = [&]() {
    bytes = 0;
    SFG_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, flag.p, incl.p, n, s));
    TmpBuf<char> tmp((int64_t)bytes, s);
    SFG_CUDA(cub::DeviceScan::InclusiveSum(tmp.p, bytes, flag.p, incl.p, n, s));
    int32_t nc = 0;
    SFG_CUDA(cudaMemcpyAsync(&nc, incl.p + n - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    SFG_CUDA(cudaStreamSynchronize(s));
    out.nchain = nc;
    out.cstart.alloc((int64_t)nc + 1);
    chain_ids_kernel<<<grid_for((int64_t)n + 1), 256, 0, s>>>(flag.p, incl.p, n, out.chain_of.p,
                                                              out.cstart.p);
    count_launch();
  };
  scan_ids();
  if (max_len > 0) {
    chain_cap_kernel<<<grid_for(n), 256, 0, s>>>(out.chain_of.p, out.cstart.p, n, max_len, flag.p);
    count_launch();
    scan_ids();
  }
  const int32_t nc = out.nchain;
  // chain levels
  TmpBuf<int> level(nc, s);
  TmpBuf<unsigned long long> counter(1, s);
  SFG_CUDA(cudaMemsetAsync(level.p, 0, sizeof(int) * (size_t)nc, s));
  SFG_CUDA(cudaMemsetAsync(counter.p, 0, sizeof(unsigned long long), s));
  {
    int per_sm = 0;
    SFG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, chain_levels_kernel, 256, 0));
    int64_t blocks = ((int64_t)nc * 32 + 255) / 256;
    const int64_t cap = (int64_t)(per_sm < 1 ? 1 : per_sm) * sm_count();
    if (blocks > cap)
      blocks = cap;
    chain_levels_kernel<<<(unsigned)blocks, 256, 0, s>>>(ptr, idx, n, dir, out.cstart.p,
                                                         out.chain_of.p, nc, level.p, counter.p);
    count_launch();
  }
  // claim order: stable sort of chains by level
  TmpBuf<int32_t> iota(nc, s), slev(nc, s);
  out.corder.alloc(nc);
  out.rank.alloc(nc);
  iota_kernel<<<grid_for(nc), 256, 0, s>>>(iota.p, nc);
  count_launch();
  bytes = 0;
  SFG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, level.p, slev.p, iota.p, out.corder.p,
                                           nc, 0, bits_for(nc + 1), s));
  {
    TmpBuf<char> tmp((int64_t)bytes, s);
    SFG_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, level.p, slev.p, iota.p,
                                             out.corder.p, nc, 0, bits_for(nc + 1), s));
  }
  SFG_CUDA(cudaMemcpyAsync(&out.nlevels, slev.p + nc - 1, sizeof(int32_t), cudaMemcpyDeviceToHost,
                           s));
  out.clevel.alloc(nc);
  SFG_CUDA(cudaMemcpyAsync(out.clevel.p, level.p, sizeof(int32_t) * (size_t)nc,
                           cudaMemcpyDeviceToDevice, s));
  // warp batches: <= CS chains of one level
  TmpBuf<int32_t> rstart(nc, s), bflag((int64_t)nc + 1, s), bid((int64_t)nc + 1, s);
  batch_flag_kernel<<<grid_for(nc), 256, 0, s>>>(slev.p, nc, CS, rstart.p);
  bytes = 0;
  SFG_CUDA(cub::DeviceScan::InclusiveScan(nullptr, bytes, rstart.p, rstart.p, cub::Max(), nc, s));
  {
    TmpBuf<char> tmp((int64_t)bytes, s);
    SFG_CUDA(cub::DeviceScan::InclusiveScan(tmp.p, bytes, rstart.p, rstart.p, cub::Max(), nc, s));
  }
  batch_flag2_kernel<<<grid_for((int64_t)nc + 1), 256, 0, s>>>(rstart.p, nc, CS, out.corder.p,
                                                               bflag.p, out.rank.p);
  bytes = 0;
  SFG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, bflag.p, bid.p, nc + 1, s));
  {
    TmpBuf<char> tmp((int64_t)bytes, s);
    SFG_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, bflag.p, bid.p, nc + 1, s));
  }
  int32_t nb = 0;
  SFG_CUDA(cudaMemcpyAsync(&nb, bid.p + nc, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  SFG_CUDA(cudaStreamSynchronize(s));
  out.nbatch = nb;
  out.batch_ptr.alloc((int64_t)nb + 1);
  batch_ptr_kernel<<<grid_for((int64_t)nc + 1), 256, 0, s>>>(bflag.p, bid.p, nc, nb,
                                                             out.batch_ptr.p);
  count_launch(3);
  out.rows_chained = n - nc;
  SFG_CUDA(cudaGetLastError());
  SFG_CUDA(cudaStreamSynchronize(s));
}

void build_tails(const ChainLayout& fwd, const int32_t* ar_ptr, const int32_t* ar_idx, int32_t n,
                 DBuf<int32_t>& tail_ptr, DBuf<int32_t>& tail_rows, cudaStream_t s) {
  const int32_t nc = fwd.nchain;
  tail_ptr.alloc((int64_t)nc + 1);
  tail_rows.alloc(n > 0 ? n : 1);
  if (n == 0) {
    SFG_CUDA(cudaMemsetAsync(tail_ptr.p, 0, sizeof(int32_t) * ((size_t)nc + 1), s));
    return;
  }
  TmpBuf<int32_t> owner(n, s), cnt((int64_t)nc + 1, s), cursor((int64_t)nc + 1, s);
  SFG_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int32_t) * ((size_t)nc + 1), s));
  tail_owner_kernel<<<grid_for(n), 256, 0, s>>>(ar_ptr, ar_idx, fwd.chain_of.p, fwd.rank.p,
                                                fwd.corder.p, n, owner.p, cnt.p);
  size_t bytes = 0;
  SFG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, cnt.p, tail_ptr.p, nc + 1, s));
  {
    TmpBuf<char> tmp((int64_t)bytes, s);
    SFG_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, cnt.p, tail_ptr.p, nc + 1, s));
  }
  SFG_CUDA(cudaMemcpyAsync(cursor.p, tail_ptr.p, sizeof(int32_t) * ((size_t)nc + 1),
                           cudaMemcpyDeviceToDevice, s));
  tail_scatter_kernel<<<grid_for(n), 256, 0, s>>>(owner.p, n, cursor.p, tail_rows.p);
  count_launch(2);
  SFG_CUDA(cudaGetLastError());
  SFG_CUDA(cudaStreamSynchronize(s));
}

void launch_chain(const ChainArgs& a, cudaStream_t s) {
  if (a.seg_end <= a.seg_begin)
    return;
  switch (a.combo) {
  case 1:
    launch_c<1>(a, s);
    break;
  case 4:
    if (a.S != 1)
      throw InvalidArgument("combo 4 supports a single system");
    launch_t<1, 4>(a, s);
    break;
  case 8:
    launch_c<8>(a, s);
    break;
  default:
    throw InvalidArgument("launch_chain: bad combo");
  }
}

} // namespace sfg
