// micro_step.cu -- cost of one carried-chain step on this GPU, with each
// ingredient toggled: the IEEE division, the relaxed.gpu publish store, the
// shuffle hand-off between lane groups, and the divergent per-group turn.
// One warp runs a chain of N steps; T/N = step cost.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void st_relaxed(void* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __noinline__ double slow_div(double v, double d) { return __ddiv_rn(v, d); }
__device__ __forceinline__ void st_plain(double* p, double v) { *p = v; }

template <int DIV, int PUB, int SHFL, int G>
__global__ void chain(double* out, const double* coef, int n, long long* cycles) {
  const int lane = threadIdx.x & 31;
  const int k = lane % G;
  double carry = 1.0, x = 0.0;
  const long long t0 = clock64();
  for (int t = 0; t < n; t += G) {
#pragma unroll 1
    for (int kk = 0; kk < G; ++kk) {
      if (k == kk) {
        const double a = coef[(t + kk) & 1023];
        const double v = __dsub_rn(a, __dmul_rn(0.5, carry));
        if (DIV == 1)
          x = __ddiv_rn(v, 1.000001);
        else if (DIV == 2) { // Markstein with a precomputed reciprocal, guarded
          const double d = 1.000001, r = 0.999999000001;
          const double av = fabs(v);
          if (!(av > 0x1p-500 && av < 0x1p+500))
            x = __ddiv_rn(v, d);
          else {
            const double q0 = __dmul_rn(v, r);
            x = __fma_rn(__fma_rn(-q0, d, v), r, q0);
          }
        } else if (DIV == 4) { // Markstein, exponent guard, out-of-line slow path
          const double d = 1.000001, r = 0.999999000001;
          const unsigned e = ((unsigned)(__double_as_longlong(v) >> 52)) & 0x7FFu;
          const double q0 = __dmul_rn(v, r);
          x = __fma_rn(__fma_rn(-q0, d, v), r, q0);
          if (__builtin_expect(e - 523u > 1000u, 0))
            x = slow_div(v, d);
        } else if (DIV == 3) { // Markstein, unguarded
          const double d = 1.000001, r = 0.999999000001;
          const double q0 = __dmul_rn(v, r);
          x = __fma_rn(__fma_rn(-q0, d, v), r, q0);
        } else
          x = __dmul_rn(v, 0.999999);
        if (PUB == 1)
          st_relaxed(out + ((t + kk) & 1023) * 32 + lane, (unsigned long long)__double_as_longlong(x));
        else if (PUB == 2)
          st_plain(out + ((t + kk) & 1023) * 32 + lane, x);
      }
      carry = SHFL ? __shfl_sync(0xffffffffu, x, kk) : x;
    }
  }
  if (lane == 0)
    cycles[0] = clock64() - t0;
  out[lane] += carry;
}

template <int DIV, int PUB, int SHFL, int G> void run(const char* name, double* out, double* coef,
                                                      long long* cyc) {
  const int n = 4096;
  chain<DIV, PUB, SHFL, G><<<1, 32>>>(out, coef, n, cyc);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  chain<DIV, PUB, SHFL, G><<<1, 32>>>(out, coef, n, cyc);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("%-40s %.1f ns/step  %.1f cycles/step\n", name, ms * 1e6 / n, (double)c / n);
}

int main() {
  double *out, *coef;
  long long* cyc;
  cudaMalloc(&out, 1024 * 32 * 8 + 256);
  cudaMalloc(&coef, 1024 * 8);
  cudaMalloc(&cyc, 8);
  { double h[1024]; for (int i = 0; i < 1024; ++i) h[i] = 0.5 + i * 1e-3; cudaMemcpy(coef, h, sizeof(h), cudaMemcpyHostToDevice); }
  run<2, 1, 1, 4>("markstein guarded + store + shfl, G=4", out, coef, cyc);
  run<3, 1, 1, 4>("markstein unguarded + store + shfl, G=4", out, coef, cyc);
  run<4, 1, 1, 4>("markstein exp-guard + noinline slow, G=4", out, coef, cyc);
  run<2, 1, 0, 1>("markstein guarded + store, G=1", out, coef, cyc);
  run<0, 1, 0, 1>("mul + store, G=1", out, coef, cyc);
  run<1, 1, 1, 8>("div + relaxed.gpu store + shfl, G=8", out, coef, cyc);
  run<1, 2, 1, 8>("div + plain store + shfl, G=8", out, coef, cyc);
  run<1, 0, 1, 8>("div + no store + shfl, G=8", out, coef, cyc);
  run<0, 1, 1, 8>("mul + relaxed.gpu store + shfl, G=8", out, coef, cyc);
  run<0, 0, 1, 8>("mul + no store + shfl, G=8", out, coef, cyc);
  run<1, 1, 1, 4>("div + relaxed.gpu store + shfl, G=4", out, coef, cyc);
  run<1, 1, 0, 1>("div + relaxed.gpu store, no shfl, G=1", out, coef, cyc);
  run<1, 0, 0, 1>("div only, G=1", out, coef, cyc);
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
