// lock.cu -- lockstep chain executor for batched solve pairs (combo 8 with
// S >= 2 interleaved systems; trsv_csr_row, kernels.hpp:171-181, forward and
// on the rows of L^T backward).
//
// A warp owns a batch of 32/S chains of ONE chain-DAG level (no chain of the
// batch depends on another), lane = (chain c, system s), and advances all of
// them one row per step.  The carry x_{p-1} of a chain therefore never leaves
// its lane's registers: no shuffles, no tile skew, and every lane works in
// every step of the recurrence.  All other operands are external (rows of
// chains of earlier levels, claimed earlier) and come through a software
// pipeline that keeps every load off the recurrence:
//   step t+DV+2  row pointers                        -> registers
//   step t+DV    values, indices, header of the row  -> shared-memory ring (cp.async)
//   step t+2     the row's dependency words and rhs  -> registers (ld.relaxed)
//   step t+1     RN(1/d)
//   step t       re-poll what is still unpublished, 12-term sum in the
//                reference order, carry term, Markstein division, publish
// The arithmetic is the reference's, term by term (separately rounded
// product and difference, ascending storage order, carry last).
#include <cstdlib>

#include "chain.cuh"
#include "common.cuh"

#ifndef SFG_LOCK_WARPS
#define SFG_LOCK_WARPS 6
#endif
#ifndef SFG_LOCK_DV
#define SFG_LOCK_DV 8 // ring depth in steps (a power of two)
#endif

namespace sfg {

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kCap = kLockTerms + 2; // staged entries per row: external terms, carry term, diagonal
#ifndef SFG_LOCK_DX
#define SFG_LOCK_DX 2
#endif
#ifndef SFG_LOCK_TRACE
#define SFG_LOCK_TRACE 1
#endif
constexpr int DX = SFG_LOCK_DX; // steps between the dependency-word loads and their use (1 or 2)

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N> __device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int S> struct alignas(16) LockSlot {
  double v[32 / S][kCap][S];
  double hd[32 / S][2][S]; // the row's diagonal and carry coefficient, at fixed places
  int32_t idx[32 / S][16];
  int32_t meta[32 / S][2]; // entries of the row (diagonal included), unused
};

// max over positions of the row's external (non-carry) dependencies
__global__ void lock_terms_kernel(const int32_t* __restrict__ ptr, int32_t n, int dir,
                                  const int32_t* __restrict__ chain_of,
                                  const int32_t* __restrict__ cstart, int32_t* out) {
  int mx = 0;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int r = dir > 0 ? (int)p : n - 1 - (int)p;
    const int cnt = ptr[r + 1] - ptr[r] - 1;
    const bool chained = cstart[chain_of[p]] != (int)p;
    mx = max(mx, cnt - (chained ? 1 : 0));
  }
  mx = __reduce_max_sync(FULL, mx);
  if ((threadIdx.x & 31) == 0)
    atomicMax(out, mx);
}

template <int S, int W, int DV>
__global__ void __launch_bounds__(W * 32, 1) k_lock(const ChainArgs A) {
  static_assert((DV & (DV - 1)) == 0 && DV > DX + 1, "ring depth");
  static_assert(S >= 2 && S % 2 == 0 && S <= 32, "pair copies need an even number of systems");
  constexpr int CS = 32 / S;
  constexpr int VR = (kCap * S / 2 + S - 1) / S; // 16-byte value chunks per lane and row
  constexpr int IR = (kCap + S - 1) / S;         // index words per lane and row
  extern __shared__ __align__(16) unsigned char smem_raw[];
  using Slot = LockSlot<S>;
  Slot* ring = reinterpret_cast<Slot*>(smem_raw) + DV * (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const int c = lane / S;
  const int s = lane % S;
  const int first_n = A.f_nbatch;
  const int total = A.seg_end - A.seg_begin;
  for (;;) {
    unsigned long long w0 = 0;
    if (lane == 0)
      w0 = atomicAdd(A.counter, 1ull);
    const long long wi = (long long)__shfl_sync(FULL, w0, 0);
    if (wi >= total)
      break;
    const int item = A.seg_begin + (int)wi;
    const bool bwd = item >= first_n;
    const int bi = bwd ? item - first_n : item;
    const int32_t* ptr = bwd ? A.lt_ptr : A.lr_ptr;
    const int32_t* idx = bwd ? A.lt_idx : A.lr_idx;
    const double* val = bwd ? A.lt_val : A.lr_val;
    const int32_t* cstart = bwd ? A.b_cstart : A.f_cstart;
    const int32_t* corder = bwd ? A.b_corder : A.f_corder;
    const int32_t* bptr = bwd ? A.b_bptr : A.f_bptr;
    double* xo = bwd ? A.vout : A.vmid;
    const double* rhs_vec = bwd ? A.vmid : A.vin;
    const int kern = bwd ? 2 : 1;
    const int q0 = __ldg(bptr + bi), q1 = __ldg(bptr + bi + 1);
    const bool has = q0 + c < q1;
    int p0 = 0, len = 0;
    if (has) {
      const int ch = __ldg(corder + q0 + c);
      p0 = __ldg(cstart + ch);
      len = __ldg(cstart + ch + 1) - p0;
    }
    const int nsteps = __reduce_max_sync(FULL, len);
    // diagnostics (SFG_TRACE): every 4th step {wait entry ns, re-poll rounds, step end ns}
    unsigned long long* tr =
        SFG_LOCK_TRACE && A.trace ? A.trace + (size_t)item * A.trace_tiles * 3 : nullptr;
    auto row_of = [&](int o) { const int p = p0 + o; return bwd ? A.n - 1 - p : p; };
    if ((A.phase & 1) && A.bwd_reset) {
      // Fused fwd -> bwd: the backward outputs are reset here (see
      // k_chain_sm): the last bwd_reset_items forward items each set one
      // slice of vout to SENT before they start; every backward item waits
      // for all slices.
      const int ri = first_n - 1 - item;
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
    if (bwd && (A.phase & 1) && A.bwd_gate) { // fused launch only
      // a backward item cannot start before the forward solve has reached
      // its first right-hand side: one lane sleeps on that word
      if (lane == 0) {
        const unsigned long long* w = reinterpret_cast<const unsigned long long*>(
            rhs_vec + (size_t)row_of(0) * S);
        while (is_sent_hi(ld_relaxed_u64(w)))
          __nanosleep(A.bwd_gate);
      }
    }
    __syncwarp();
    // register sets by step parity: dependency words, rhs word, row pointers
    unsigned long long xxA[kLockTerms], xxB[kLockTerms];
    unsigned long long rhA = 0, rhB = 0;
    int pbA = 0, peA = 0, pbB = 0, peB = 0;
    double xprev = 0.0, rd = 1.0;
#pragma unroll
    for (int a = 0; a < kLockTerms; ++a)
      xxA[a] = xxB[a] = 0;
    // header of the row the next step finishes, read one step early: entry
    // count, diagonal, carry coefficient, RN(1/diagonal)
    int cntc = 1;
    double dc = 1.0, vcc = 0.0;
    const unsigned ulen = has ? (unsigned)len : 0u;
    auto act = [&](int o) { return (unsigned)o < ulen; };
    double* const xos = xo + s;
    auto body = [&](const int t, unsigned long long(&xx)[kLockTerms], unsigned long long& rh,
                    int& pb, int& pe) {
      // every copy of steps <= t + DX has landed
      const long long ckA = tr ? clock64() : 0;
      cp_async_wait<DV - 1 - DX>();
      __syncwarp();
      const long long ckB = tr ? clock64() : 0;
      long long ckD = ckB;
      const Slot& sl = ring[t & (DV - 1)];
      const Slot& s1 = ring[(t + 1) & (DV - 1)];
      const Slot& sx = ring[(t + DX) & (DV - 1)];
      const int u = t + DX;
      const bool a0 = act(t), a1 = act(t + 1), a2 = act(u);
      // ---- every shared-memory read of this iteration, ahead of the asm
      // loads and stores (compiler barriers), so they issue back to back
      double v[kLockTerms];
#pragma unroll
      for (int a = 0; a < kLockTerms; ++a)
        v[a] = sl.v[c][a][s];
      int jx[16];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const int4 j4 = *reinterpret_cast<const int4*>(&sx.idx[c][4 * k]);
        jx[4 * k] = j4.x, jx[4 * k + 1] = j4.y, jx[4 * k + 2] = j4.z, jx[4 * k + 3] = j4.w;
      }
      const int mu = a2 ? sx.meta[c][0] - 1 - (u > 0 ? 1 : 0) : 0;
      const int cnt1 = s1.meta[c][0];
      const double d1 = s1.hd[c][0][s];
      const double vc1 = t + 1 > 0 ? s1.hd[c][1][s] : 0.0; // no carry into a chain's first row
      // ---- step t: finish the row
      if (a0) {
        const int m = cntc - 1 - (t > 0 ? 1 : 0);
        const int r = row_of(t);
        const bool trs = tr && lane == 0 && (t & 3) == 0 && (t >> 2) < A.trace_tiles;
        unsigned long long rounds = 0;
        if (trs)
          tr[(t >> 2) * 3] = gtimer();
        double acc;
        if (m == kLockTerms) { // full-width row: no per-term predicates
          for (;;) {
            unsigned hi = bwd ? (unsigned)(rh >> 32) : 0u;
#pragma unroll
            for (int a = 0; a < kLockTerms; ++a)
              hi = max(hi, (unsigned)(xx[a] >> 32));
            if (hi != 0xFFFFFFFFu)
              break;
            ++rounds;
            if (A.poll_ns)
              __nanosleep(A.poll_ns);
            if (bwd && is_sent_hi(rh))
              rh = ld_relaxed_u64(rhs_vec + (size_t)r * S + s);
#pragma unroll
            for (int a = 0; a < kLockTerms; ++a)
              if (is_sent_hi(xx[a]))
                xx[a] = ld_relaxed_u64(xos + (size_t)sl.idx[c][a] * S);
          }
          acc = __longlong_as_double((long long)rh);
#pragma unroll
          for (int a = 0; a < kLockTerms; ++a)
            acc = __dsub_rn(acc, __dmul_rn(v[a], __longlong_as_double((long long)xx[a])));
        } else {
          for (;;) {
            bool pending = bwd && is_sent_hi(rh);
#pragma unroll
            for (int a = 0; a < kLockTerms; ++a)
              pending |= a < m && is_sent_hi(xx[a]);
            if (!pending)
              break;
            ++rounds;
            if (A.poll_ns)
              __nanosleep(A.poll_ns);
            if (bwd && is_sent_hi(rh))
              rh = ld_relaxed_u64(rhs_vec + (size_t)r * S + s);
#pragma unroll
            for (int a = 0; a < kLockTerms; ++a)
              if (a < m && is_sent_hi(xx[a]))
                xx[a] = ld_relaxed_u64(xos + (size_t)sl.idx[c][a] * S);
          }
          acc = __longlong_as_double((long long)rh);
#pragma unroll
          for (int a = 0; a < kLockTerms; ++a)
            if (a < m)
              acc = __dsub_rn(acc, __dmul_rn(v[a], __longlong_as_double((long long)xx[a])));
        }
        // the carry term, last in the reference order (first row of a chain:
        // vcc = +0 and xprev = +0, and acc - (+0) == acc for every acc)
        acc = __dsub_rn(acc, __dmul_rn(vcc, xprev));
        if (dc == 0.0)
          report_error(A.err, kern, bwd ? A.n - 1 - r : r, r);
        const double q0d = __dmul_rn(acc, rd);
        double q = __fma_rn(__fma_rn(-q0d, dc, acc), rd, q0d);
        if (__builtin_expect(!(exp_in_safe_range(acc) && exp_in_safe_range(dc)), 0))
          q = ieee_div_slow(acc, dc);
        publish_f64(xos + (size_t)r * S, q);
        xprev = q;
        if (trs) {
          tr[(t >> 2) * 3 + 1] = rounds;
          tr[(t >> 2) * 3 + 2] = gtimer();
          ckD = clock64();
        }
      }
      // ---- step t + DX: dependency words and right-hand side
      if (a2) {
        const int ru = row_of(u);
        rh = bwd ? ld_relaxed_u64(rhs_vec + (size_t)ru * S + s)
                 : (unsigned long long)__double_as_longlong(__ldg(rhs_vec + (size_t)ru * S + s));
        if (mu == kLockTerms) {
#pragma unroll
          for (int a = 0; a < kLockTerms; ++a)
            xx[a] = ld_relaxed_u64(xos + (size_t)jx[a] * S);
        } else {
#pragma unroll
          for (int a = 0; a < kLockTerms; ++a)
            if (a < mu)
              xx[a] = ld_relaxed_u64(xos + (size_t)jx[a] * S);
        }
      }
      // ---- step t + 1: its header, and the reciprocal of its diagonal
      cntc = cnt1;
      dc = d1;
      vcc = vc1;
      rd = a1 ? __drcp_rn(d1) : 1.0;
      __syncwarp(); // slot t is free: every lane has read it
      // ---- step t + DV: stage the row
      {
        const int w = t + DV;
        if (act(w)) {
          Slot& sv = ring[w & (DV - 1)];
          const int cnt = pe - pb;
          if (s == 0)
            sv.meta[c][0] = cnt;
          const double* src = val + (size_t)pb * S + 2 * s;
          double* dst = &sv.v[c][0][0] + 2 * s;
          const int nchunk = cnt * (S / 2) - s;
#pragma unroll
          for (int k = 0; k < VR; ++k)
            if (k * S < nchunk)
              cp_async16(dst + 2 * k * S, src + 2 * k * S);
          if ((s & 1) == 0) { // header: the diagonal and the entry before it
            cp_async16(&sv.hd[c][0][s], val + (size_t)(pe - 1) * S + s);
            if (cnt >= 2)
              cp_async16(&sv.hd[c][1][s], val + (size_t)(pe - 2) * S + s);
          }
#pragma unroll
          for (int k = 0; k < IR; ++k) {
            const int e = s + k * S;
            if (e < cnt - 1)
              cp_async4(&sv.idx[c][e], idx + pb + e);
          }
        }
        cp_async_commit();
      }
      // ---- step t + DV + 2: row pointers
      {
        const int z = t + DV + 2;
        if (act(z)) {
          const int rz = row_of(z);
          pb = __ldg(ptr + rz);
          pe = __ldg(ptr + rz + 1);
        }
      }
      if (tr && a0 && lane == 0 && (t & 3) == 0 && (t >> 2) < A.trace_tiles) {
        // rounds | cycles in the copy wait | wait end -> published | published -> end of body
        auto f16 = [](long long x) { return (unsigned long long)(x < 0 ? 0 : (x > 65535 ? 65535 : x)); };
        tr[(t >> 2) * 3 + 1] = (tr[(t >> 2) * 3 + 1] & 0xFFFF) | (f16(ckB - ckA) << 16) |
                               (f16(ckD - ckB) << 32) | (f16(clock64() - ckD) << 48);
      }
    };
#pragma unroll 1
    for (int t = -(DV + 2); t < nsteps; t += 2) {
      body(t, xxA, rhA, pbA, peA);
      if (DX == 2)
        body(t + 1, xxB, rhB, pbB, peB);
      else
        body(t + 1, xxA, rhA, pbB, peB);
    }
    cp_async_wait<0>();
    __syncwarp();
  }
}

constexpr int lock_warps(size_t slot, int dv) {
  int w = SFG_LOCK_WARPS;
  while (w > 1 && (size_t)w * dv * slot > 227u * 1024u)
    --w;
  return w;
}

template <int S> void launch_s(const ChainArgs& a, cudaStream_t s) {
  constexpr int DV = SFG_LOCK_DV;
  constexpr int W = lock_warps(sizeof(LockSlot<S>), DV);
  auto kern = k_lock<S, W, DV>;
  const size_t smem = (size_t)W * DV * sizeof(LockSlot<S>);
  SFG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t items = a.seg_end - a.seg_begin;
  int64_t grid = (items + W - 1) / W;
  if (grid > sm_count())
    grid = sm_count();
  static const int grid_cap = getenv("SFG_LOCK_GRID") ? atoi(getenv("SFG_LOCK_GRID")) : 0;
  if (grid_cap > 0 && grid > grid_cap) // diagnostics: fewer CTAs (1 = no contention)
    grid = grid_cap;
  if (grid < 1)
    return;
  kern<<<(unsigned)grid, W * 32, smem, s>>>(a);
  count_launch();
  SFG_CUDA(cudaGetLastError());
}

} // namespace

int32_t lock_max_terms(const int32_t* ptr, int32_t n, int dir, const ChainLayout& L,
                       cudaStream_t s) {
  if (n == 0)
    return 0;
  DBuf<int32_t> out(1);
  SFG_CUDA(cudaMemsetAsync(out.p, 0, sizeof(int32_t), s));
  int64_t g = ((int64_t)n + 255) / 256;
  if (g > (int64_t)sm_count() * 8)
    g = (int64_t)sm_count() * 8;
  lock_terms_kernel<<<(unsigned)g, 256, 0, s>>>(ptr, n, dir, L.chain_of.p, L.cstart.p, out.p);
  count_launch();
  int32_t h = 0;
  SFG_CUDA(cudaMemcpyAsync(&h, out.p, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  SFG_CUDA(cudaStreamSynchronize(s));
  return h;
}

void launch_lock(const ChainArgs& a, cudaStream_t s) {
  if (a.seg_end <= a.seg_begin)
    return;
  if (a.combo != 8)
    throw InvalidArgument("launch_lock: the lockstep executor runs combo 8");
  switch (a.S) {
  case 2:
    launch_s<2>(a, s);
    break;
  case 4:
    launch_s<4>(a, s);
    break;
  case 8:
    launch_s<8>(a, s);
    break;
  case 16:
    launch_s<16>(a, s);
    break;
  case 32:
    launch_s<32>(a, s);
    break;
  default:
    throw InvalidArgument("launch_lock: nsys must be a power of two in 2..32");
  }
}

} // namespace sfg
