// selftest.cu -- device-side checks exposed through the C-ABI.
#include "../../include/sfgpu.h"
#include "common.cuh"
#include "internal.hpp"

namespace sfg {
namespace {

__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Random operands: uniform mantissas, exponents drawn from a wide range so
// both the fast path and the guarded fallback are exercised; every 16th pair
// uses solver-like magnitudes (|v| ~ 1e-3..1e3, d ~ 1..64).
__global__ void div_check_kernel(long long n, unsigned long long seed,
                                 unsigned long long* mismatches, unsigned long long* fast) {
  unsigned long long bad = 0, fp = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const unsigned long long h1 = mix64(seed ^ (unsigned long long)i);
    const unsigned long long h2 = mix64(h1);
    const unsigned long long h3 = mix64(h2);
    double v, d;
    if ((i & 15) == 0) {
      v = ((double)(h1 >> 11) * 0x1p-53 * 2.0 - 1.0) * exp2((double)((int)(h3 % 21) - 10));
      d = 1.0 + (double)(h2 >> 11) * 0x1p-53 * 63.0;
    } else {
      const int ev = (int)(h3 % 1200) - 600, ed = (int)((h3 >> 16) % 1200) - 600;
      v = __longlong_as_double((long long)(((h1 & 0x000FFFFFFFFFFFFFull) |
                                            ((unsigned long long)(ev + 1023) << 52)) |
                                           (h1 & 0x8000000000000000ull)));
      d = __longlong_as_double((long long)(((h2 & 0x000FFFFFFFFFFFFFull) |
                                            ((unsigned long long)(ed + 1023) << 52)) |
                                           (h2 & 0x8000000000000000ull)));
    }
    const double want = __ddiv_rn(v, d);
    const double got = div_with_rcp(v, d, __drcp_rn(d));
    if (exp_in_safe_range(v) && exp_in_safe_range(d))
      ++fp;
    if (__double_as_longlong(want) != __double_as_longlong(got))
      ++bad;
  }
  atomicAdd(mismatches, bad);
  atomicAdd(fast, fp);
}

} // namespace
} // namespace sfg

extern "C" sfg_status sfg_selftest_division(int64_t n, uint64_t seed, int64_t* mismatches,
                                            int64_t* fast_path) {
  using namespace sfg;
  int cnt = 0;
  if (cudaGetDeviceCount(&cnt) != cudaSuccess || cnt <= 0) {
    cudaGetLastError();
    return SFG_ERR_NO_DEVICE;
  }
  unsigned long long* d = nullptr;
  if (cudaMalloc(&d, 2 * sizeof(unsigned long long)) != cudaSuccess)
    return SFG_ERR_CUDA;
  cudaMemset(d, 0, 2 * sizeof(unsigned long long));
  div_check_kernel<<<sm_count() * 8, 256>>>(n, seed, d, d + 1);
  unsigned long long h[2] = {0, 0};
  const cudaError_t e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess)
    return SFG_ERR_CUDA;
  if (mismatches)
    *mismatches = (int64_t)h[0];
  if (fast_path)
    *fast_path = (int64_t)h[1];
  return SFG_OK;
}
