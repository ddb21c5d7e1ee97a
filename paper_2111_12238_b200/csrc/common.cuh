// common.cuh -- device-side building blocks shared by the inspector and the
// executor kernels (sm_100a only).
//
// Synchronisation model (replaces SpinBarrier + std::atomic claims of
// executor.hpp:36-68,416-456).  Every value one task produces for another is
// a 64-bit word that is reset to SENT (all-ones, a NaN no IEEE operation
// produces from non-SENT operands) before the launch.  A consumer polls the
// very word it needs with ld.relaxed.gpu until it is not SENT; the producer
// writes it once with st.relaxed.gpu.  Because each polled word is its own
// flag there is no separate flag array, no fence and no second L2 round trip
// per dependency.  Work is claimed as warp-wide tickets from one global
// counter in a topological order, so every task a warp waits on has already
// been claimed by a running warp: sync-free and deadlock-free without
// relying on CTA residency.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace sfg {

constexpr unsigned long long SENT = 0xFFFFFFFFFFFFFFFFull;
constexpr unsigned long long CANON_NAN = 0x7FF8000000000000ull;

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const void* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Read-only (non-coherent) load pinned in program order (asm volatile), so
// the compiler cannot hoist it across the executor's wait loops.
__device__ __forceinline__ double ld_nc_f64(const double* p) {
  double v;
  asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ void st_relaxed_u64(void* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ int ld_relaxed_i32(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_relaxed_i32(int* p, int v) {
  asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Spin until *p is published (high word not all-ones, see publish_f64); an optional exponential nanosleep backoff (capped at
// g_sleep_cap ns; 0 = pure spin) keeps pollers off the producers' L2 slices.
__device__ __forceinline__ double poll_f64(const double* p, unsigned sleep_cap = 160) {
  unsigned long long v = ld_relaxed_u64(p);
  if ((unsigned)(v >> 32) != 0xFFFFFFFFu)
    return __longlong_as_double((long long)v);
  unsigned ns = 20;
  do {
    if (sleep_cap) {
      __nanosleep(ns);
      ns = ns < sleep_cap ? ns * 2 : sleep_cap;
    }
    v = ld_relaxed_u64(p);
  } while ((unsigned)(v >> 32) == 0xFFFFFFFFu);
  return __longlong_as_double((long long)v);
}

// Publish a value.  Every NaN is stored as the canonical quiet NaN, so no
// published word -- and no finite value -- has an all-ones high word: a
// consumer can test readiness on the high 32 bits alone (is_sent_hi).
__device__ __forceinline__ void publish_f64(double* p, double v) {
  unsigned long long b = (unsigned long long)__double_as_longlong(v);
  if (v != v)
    b = CANON_NAN;
  st_relaxed_u64(p, b);
}

__device__ __forceinline__ bool is_sent_hi(unsigned long long w) {
  return (unsigned)(w >> 32) == 0xFFFFFFFFu;
}

// Integer flavour for the inspector: 0 = not ready (levels are >= 1).
__device__ __forceinline__ int poll_pos_i32(const int* p) {
  int v = ld_relaxed_i32(p);
  if (v > 0)
    return v;
  unsigned ns = 20;
  do {
    __nanosleep(ns);
    ns = ns < 160 ? ns * 2 : 160;
    v = ld_relaxed_i32(p);
  } while (v <= 0);
  return v;
}

// Heights use -1 as "not ready" (heights are >= 0).
__device__ __forceinline__ int poll_nonneg_i32(const int* p) {
  int v = ld_relaxed_i32(p);
  if (v >= 0)
    return v;
  unsigned ns = 20;
  do {
    __nanosleep(ns);
    ns = ns < 160 ? ns * 2 : 160;
    v = ld_relaxed_i32(p);
  } while (v < 0);
  return v;
}

// Warp-granular ticket claim: lane 0 takes `per_warp` tickets, broadcast.
__device__ __forceinline__ long long claim_tickets(unsigned long long* counter,
                                                   int per_warp) {
  unsigned long long base = 0;
  if ((threadIdx.x & 31) == 0)
    base = atomicAdd(counter, (unsigned long long)per_warp);
  return (long long)__shfl_sync(0xffffffffu, base, 0);
}

// Error word: the minimum key over all failing tasks reproduces the first
// failure of the sequential reference (run_sequential_reference runs every
// kernel-1 iteration before kernel 2, ascending): key = kernel-1 (bit 62) |
// sequential position of the detecting iteration (bits 31..61) | index.
__device__ __forceinline__ void report_error(unsigned long long* word,
                                             int kernel, int seq_pos,
                                             int index) {
  const unsigned long long key =
      ((unsigned long long)(kernel - 1) << 62) |
      ((unsigned long long)(unsigned)seq_pos << 31) | (unsigned)index;
  atomicMin(word, key);
}

// Correctly rounded v / d given r = RN(1/d) computed earlier (off the
// critical path): q0 = RN(v r), rho = v - q0 d (exact with FMA), q = RN(q0 +
// rho r) -- Markstein's correction, which returns RN(v / d) when r is the
// correctly rounded reciprocal and no intermediate leaves the normal range.
// Operands near the exponent limits, zeros, infinities and NaNs take the
// IEEE division itself, so the result always equals __ddiv_rn(v, d)
// (checked by sfg_selftest_division over random operands).
static __device__ __noinline__ double ieee_div_slow(double v, double d) { return __ddiv_rn(v, d); }

// biased exponent of |x| inside [2^-500, 2^500): 523 <= e <= 1522
__device__ __forceinline__ bool exp_in_safe_range(double x) {
  const unsigned e = (unsigned)((unsigned long long)__double_as_longlong(x) >> 52) & 0x7FFu;
  return e - 523u < 1000u;
}

__device__ __forceinline__ double div_with_rcp(double v, double d, double r) {
  const double q0 = __dmul_rn(v, r);
  const double q = __fma_rn(__fma_rn(-q0, d, v), r, q0);
  if (__builtin_expect(!(exp_in_safe_range(v) && exp_in_safe_range(d)), 0))
    return ieee_div_slow(v, d);
  return q;
}

__device__ __forceinline__ double ldg_f64(const double* p) { return __ldg(p); }
__device__ __forceinline__ int ldg_i32(const int* p) { return __ldg(p); }

} // namespace sfg
