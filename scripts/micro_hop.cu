// micro_hop.cu -- measures the cost of one dependent hop through global
// memory on this GPU: task t (claimed in ticket order by some warp) waits
// for task t-1's word, then publishes its own.  T / ntasks = hop latency.
// Variants: spin vs nanosleep backoff; tasks handled by separate warps
// (dynamic tickets) vs a dependent chain inside one thread.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long ldr(const void* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void str(void* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ldv(const void* p) {
  unsigned long long v;
  asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// stride: tasks t and t-1 spaced `stride` words apart; width: how many
// independent chains run side by side (tickets interleaved)
template <int SLEEP, int VOL>
__global__ void chain(unsigned long long* words, int ntasks, int width, int stride,
                      unsigned long long* counter) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    unsigned long long base = 0;
    if (lane == 0)
      base = atomicAdd(counter, 32ull);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (base >= (unsigned long long)ntasks * width)
      break;
    const long long t = base + lane;
    if (t >= (long long)ntasks * width)
      continue;
    const long long step = t / width, c = t % width;
    unsigned long long v = 1;
    if (step > 0) {
      const unsigned long long* src = words + ((step - 1) * width + c) * stride;
      unsigned ns = 20;
      for (;;) {
        v = VOL ? ldv(src) : ldr(src);
        if (v != ~0ull)
          break;
        if (SLEEP) {
          __nanosleep(ns);
          ns = ns < 160 ? ns * 2 : 160;
        }
      }
      v += 1;
    }
    str(words + (step * width + c) * stride, v);
  }
}

int main(int argc, char** argv) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int ntasks = 4096;
  unsigned long long *words, *counter;
  const size_t maxw = (size_t)ntasks * 4096 * 8;
  cudaMalloc(&words, maxw * 8);
  cudaMalloc(&counter, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int widths[] = {1, 32, 1024, 4096};
  for (int variant = 0; variant < 3; ++variant) {
    for (int wi = 0; wi < 4; ++wi) {
      const int width = widths[wi];
      const int stride = 8; // one 64-byte segment per task
      for (int blocks_per_sm = 1; blocks_per_sm <= 8; blocks_per_sm *= 8) {
        float best = 1e30f;
        for (int rep = 0; rep < 3; ++rep) {
          cudaMemset(words, 0xFF, (size_t)ntasks * width * stride * 8);
          cudaMemset(counter, 0, 8);
          cudaEventRecord(a);
          if (variant == 0)
            chain<1, 0><<<sms * blocks_per_sm, 256>>>(words, ntasks, width, stride, counter);
          else if (variant == 1)
            chain<0, 0><<<sms * blocks_per_sm, 256>>>(words, ntasks, width, stride, counter);
          else
            chain<0, 1><<<sms * blocks_per_sm, 256>>>(words, ntasks, width, stride, counter);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          if (ms < best)
            best = ms;
        }
        printf("variant=%s width=%5d blocks/SM=%d  %.3f ms  hop=%.1f ns  (%.2f Gtask/s)\n",
               variant == 0 ? "relaxed+sleep" : variant == 1 ? "relaxed+spin " : "volatile+spin",
               width, blocks_per_sm, best, best * 1e6 / ntasks,
               (double)ntasks * width / (best * 1e-3) / 1e9);
      }
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
