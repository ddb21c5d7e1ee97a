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

#ifndef SFG_LOCK_PAIRS
#define SFG_LOCK_PAIRS 6 // warp pairs (compute + feeder) per CTA, one CTA per SM
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

// ---- mbarrier helpers (shared::cta, 64-bit objects) -----------------------
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(b);
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(b);
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared.b64 st, [%0];\n\t}" ::"r"(a) : "memory");
}
// arrives once every cp.async this thread issued before has landed
__device__ __forceinline__ void mbar_arrive_cp_async(unsigned long long* b) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(b);
  asm volatile("cp.async.mbarrier.arrive.noinc.shared.b64 [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(b);
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n\t"
      "@p bra DONE;\n\t"
      "bra LAB_WAIT;\n\t"
      "DONE:\n\t}" ::"r"(a), "r"(parity) : "memory");
}
__device__ __forceinline__ void pair_sync(int id) { // the two warps of a pair
  asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory");
}

// One pair of warps per batch of 32/S same-level chains.  The FEEDER warp
// stages each step's row (values, indices, header) into the pair's
// shared-memory ring, up to DV steps ahead, and signals full[slot] through
// the copies' own completion (cp.async.mbarrier.arrive).  The COMPUTE warp
// finishes one row of every chain per step -- dependency words loaded one
// step ahead straight into registers, re-polled while unpublished -- and
// hands the slot back through empty[slot].
template <int S, int NP, int DV>
__global__ void __launch_bounds__(NP * 64, 1) k_lock(const ChainArgs A) {
  static_assert((DV & (DV - 1)) == 0 && DV >= 2, "ring depth");
  static_assert(S >= 2 && S % 2 == 0 && S <= 32, "pair copies need an even number of systems");
  constexpr int CS = 32 / S;
  constexpr int VR = (kCap * S / 2 + S - 1) / S; // 16-byte value chunks per lane and row
  constexpr int IR = (kCap + S - 1) / S;         // index words per lane and row
  extern __shared__ __align__(16) unsigned char smem_raw[];
  using Slot = LockSlot<S>;
  const int pair = threadIdx.x >> 6;
  const bool feeder = (threadIdx.x >> 5) & 1;
  Slot* ring = reinterpret_cast<Slot*>(smem_raw) + DV * pair;
  unsigned long long* bars =
      reinterpret_cast<unsigned long long*>(smem_raw + sizeof(Slot) * DV * NP) + (2 * DV + 2) * pair;
  unsigned long long* full = bars;        // [DV] feeder -> compute
  unsigned long long* empty = bars + DV;  // [DV] compute -> feeder
  volatile long long* mail = reinterpret_cast<volatile long long*>(bars + 2 * DV); // claimed item
  const int lane = threadIdx.x & 31;
  const int c = lane / S;
  const int s = lane % S;
  const int first_n = A.f_nbatch;
  const int total = A.seg_end - A.seg_begin;
  if (!feeder && lane == 0) {
    for (int k = 0; k < DV; ++k) {
      mbar_init(full + k, 32);
      mbar_init(empty + k, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  pair_sync(1 + pair);
  unsigned g = 0; // steps this pair has run: slot = g mod DV, phase = (g / DV) & 1
  for (;;) {
    if (!feeder && lane == 0)
      *mail = (long long)atomicAdd(A.counter, 1ull);
    pair_sync(1 + pair);
    const long long wi = *mail;
    pair_sync(1 + pair); // both warps have read the mailbox
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
    const unsigned ulen = has ? (unsigned)len : 0u;
    auto act = [&](int o) { return (unsigned)o < ulen; };
    auto row_of = [&](int o) { const int p = p0 + o; return bwd ? A.n - 1 - p : p; };
    if (feeder) {
      // ---- feeder: row pointers two steps ahead, then the row's copies
      int pbA = 0, peA = 0, pbB = 0, peB = 0;
      auto fetch = [&](int z, int& pb, int& pe) {
        if (act(z)) {
          const int rz = row_of(z);
          pb = __ldg(ptr + rz);
          pe = __ldg(ptr + rz + 1);
        }
      };
      auto stage = [&](int w, int pb, int pe) {
        const unsigned gw = g + (unsigned)w;
        const int sl = gw & (DV - 1);
        mbar_wait(empty + sl, ((gw / DV) & 1) ^ 1);
        if (act(w)) {
          Slot& sv = ring[sl];
          const int cnt = pe - pb;
          if (s == 0) {
            sv.meta[c][0] = cnt;
            __threadfence_block(); // ordered before this lane's arrival below
          }
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
        mbar_arrive_cp_async(full + sl);
      };
      fetch(0, pbA, peA);
      fetch(1, pbB, peB);
#pragma unroll 1
      for (int w = 0; w < nsteps; w += 2) {
        stage(w, pbA, peA);
        fetch(w + 2, pbA, peA);
        if (w + 1 < nsteps) {
          stage(w + 1, pbB, peB);
          fetch(w + 3, pbB, peB);
        }
      }
    } else {
      // ---- compute warp
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
        if (lane == 0) {
          const unsigned long long* w = reinterpret_cast<const unsigned long long*>(
              rhs_vec + (size_t)row_of(0) * S);
          while (is_sent_hi(ld_relaxed_u64(w)))
            __nanosleep(A.bwd_gate);
        }
      }
      __syncwarp();
      double* const xos = xo + s;
      // register sets by step parity: dependency words and right-hand side
      unsigned long long xxA[kLockTerms], xxB[kLockTerms];
      unsigned long long rhA = 0, rhB = 0;
#pragma unroll
      for (int a = 0; a < kLockTerms; ++a)
        xxA[a] = xxB[a] = 0;
      double xprev = 0.0;
      // header of the row being finished / of the next one: entry count,
      // diagonal, carry coefficient, RN(1/diagonal)
      int cntc = 1, cntn = 1;
      double dc = 1.0, vcc = 0.0, rdc = 1.0, dn = 1.0, vcn = 0.0, rdn = 1.0;
      // step u's header and the loads of its operands (its slot is full)
      auto prefetch = [&](int u, unsigned long long(&xx)[kLockTerms], unsigned long long& rh) {
        const unsigned gu = g + (unsigned)u;
        mbar_wait(full + (gu & (DV - 1)), (gu / DV) & 1);
        const Slot& sx = ring[gu & (DV - 1)];
        int jx[12];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const int4 j4 = *reinterpret_cast<const int4*>(&sx.idx[c][4 * k]);
          jx[4 * k] = j4.x, jx[4 * k + 1] = j4.y, jx[4 * k + 2] = j4.z, jx[4 * k + 3] = j4.w;
        }
        const bool au = act(u);
        cntn = sx.meta[c][0];
        dn = sx.hd[c][0][s];
        vcn = u > 0 ? sx.hd[c][1][s] : 0.0; // no carry into a chain's first row
        const int mu = au ? cntn - 1 - (u > 0 ? 1 : 0) : 0;
        if (au) {
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
        rdn = au ? __drcp_rn(dn) : 1.0;
      };
      auto step = [&](int t, unsigned long long(&xx)[kLockTerms], unsigned long long& rh,
                      unsigned long long(&xxn)[kLockTerms], unsigned long long& rhn) {
        const unsigned gt = g + (unsigned)t;
        const Slot& sl = ring[gt & (DV - 1)];
        // the next step's operands go out first: they land while this row is finished
        if (t + 1 < nsteps)
          prefetch(t + 1, xxn, rhn);
        double v[kLockTerms];
#pragma unroll
        for (int a = 0; a < kLockTerms; ++a)
          v[a] = sl.v[c][a][s];
        if (act(t)) {
          const int m = cntc - 1 - (t > 0 ? 1 : 0);
          const int r = row_of(t);
          double acc;
          if (m == kLockTerms) { // full-width row: no per-term predicates
            for (;;) {
              unsigned hi = bwd ? (unsigned)(rh >> 32) : 0u;
#pragma unroll
              for (int a = 0; a < kLockTerms; ++a)
                hi = max(hi, (unsigned)(xx[a] >> 32));
              if (hi != 0xFFFFFFFFu)
                break;
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
          // the carry term, last in the reference order (first row of a
          // chain: vcc = +0, xprev = +0, and acc - (+0) == acc for every acc)
          acc = __dsub_rn(acc, __dmul_rn(vcc, xprev));
          if (dc == 0.0)
            report_error(A.err, kern, bwd ? A.n - 1 - r : r, r);
          const double q0d = __dmul_rn(acc, rdc);
          double q = __fma_rn(__fma_rn(-q0d, dc, acc), rdc, q0d);
          if (__builtin_expect(!(exp_in_safe_range(acc) && exp_in_safe_range(dc)), 0))
            q = ieee_div_slow(acc, dc);
          publish_f64(xos + (size_t)r * S, q);
          xprev = q;
        }
        __syncwarp(); // every lane is done with slot t
        if (lane == 0)
          mbar_arrive(empty + (gt & (DV - 1)));
        cntc = cntn, dc = dn, vcc = vcn, rdc = rdn;
      };
      prefetch(0, xxA, rhA);
      cntc = cntn, dc = dn, vcc = vcn, rdc = rdn;
#pragma unroll 1
      for (int t = 0; t < nsteps; t += 2) {
        step(t, xxA, rhA, xxB, rhB);
        if (t + 1 < nsteps)
          step(t + 1, xxB, rhB, xxA, rhA);
      }
    }
    g += (unsigned)nsteps;
  }
}

template <int S> void launch_s(const ChainArgs& a, cudaStream_t s) {
  constexpr int DV = SFG_LOCK_DV;
  constexpr size_t per_pair = sizeof(LockSlot<S>) * DV + (2 * DV + 2) * 8;
  constexpr int NPmax = (int)((227u * 1024u) / per_pair);
  constexpr int NP = NPmax < SFG_LOCK_PAIRS ? (NPmax < 1 ? 1 : NPmax) : SFG_LOCK_PAIRS;
  auto kern = k_lock<S, NP, DV>;
  const size_t smem = per_pair * NP;
  SFG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t items = a.seg_end - a.seg_begin;
  int64_t grid = (items + NP - 1) / NP;
  if (grid > sm_count())
    grid = sm_count();
  static const int grid_cap = getenv("SFG_LOCK_GRID") ? atoi(getenv("SFG_LOCK_GRID")) : 0;
  if (grid_cap > 0 && grid > grid_cap) // diagnostics: fewer CTAs (1 = no contention)
    grid = grid_cap;
  if (grid < 1)
    return;
  kern<<<(unsigned)grid, NP * 64, smem, s>>>(a);
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
