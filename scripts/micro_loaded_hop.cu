// Microbenchmark: one global-memory ping-pong hop (st.relaxed.gpu / poll with
// ld.relaxed.gpu) between warp 0 of CTA 0 and warp 0 of CTA `peer`, while the
// other warps of the grid stream HBM -- the loaded-L2 round trip that sets the
// per-level lag of the chain executor.
// mode 0: no background traffic; 1: cp.async.cg 16-byte streaming (as
// k_chain_sm stages values); 2: ld.global.nc streaming; 3: streaming + every
// background warp also spins ld.relaxed on a private L2 word (poll traffic).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o micro_loaded_hop micro_loaded_hop.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long ldr(const void* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void str(void* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void k_hop(int iters, int peer, int mode, int inflight, unsigned long long* words,
                      const double* big, size_t big_n, volatile int* stop, unsigned long long* out,
                      double* sink) {
  __shared__ __align__(16) double stage[16][32][8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool pinger = warp == 0 && (blockIdx.x == 0 || blockIdx.x == peer);
  if (pinger) {
    unsigned long long t0 = gtimer();
    if (lane == 0) {
      unsigned long long* mine = words + (blockIdx.x == 0 ? 0 : 32);
      unsigned long long* other = words + (blockIdx.x == 0 ? 32 : 0);
      for (unsigned long long it = 1; it <= (unsigned long long)iters; ++it) {
        if (blockIdx.x == 0) {
          str(other, 2 * it - 1);
          while (ldr(mine) != 2 * it) {
          }
        } else {
          while (ldr(mine) != 2 * it - 1) {
          }
          str(other, 2 * it);
        }
      }
    }
    __syncwarp();
    if (lane == 0 && blockIdx.x == 0) {
      out[0] = gtimer() - t0;
      *stop = 1;
    }
    return;
  }
  if (mode == 0)
    return;
  // background streaming until the ping-pong is over
  const size_t gw = (size_t)blockIdx.x * (blockDim.x >> 5) + warp;
  const size_t nw = (size_t)gridDim.x * (blockDim.x >> 5);
  size_t pos = gw * 32 * 2 * inflight;
  double acc = 0.0;
  unsigned long long* myword = words + 64 + gw * 8;
  unsigned long long rounds = 0;
  while (*stop == 0) {
    ++rounds;
    if (mode >= 4) {
      // 12 relaxed L2 loads per lane in flight (a waiting chain warp's poll
      // round), on words nobody writes; mode 5 adds the value streaming
      unsigned long long w = 0;
      const unsigned long long* base = words + 4096 + ((gw * 97 + rounds * 13) % 4096) * 64;
#pragma unroll
      for (int a = 0; a < 12; ++a)
        w += ldr(base + ((lane * 8 + a * 512 + 64) % 65536));
      acc += (double)w;
      if (mode == 5) {
        for (int f = 0; f < inflight; ++f) {
          const double* src = big + ((pos + (size_t)f * 64 + lane * 2) % big_n);
          unsigned sa = (unsigned)__cvta_generic_to_shared(&stage[warp][lane][(f & 3) * 2]);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(src) : "memory");
        }
        asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
        acc += stage[warp][lane][0];
      }
    } else if (mode == 1 || mode == 3) {
      for (int f = 0; f < inflight; ++f) {
        const double* src = big + ((pos + (size_t)f * 64 + lane * 2) % big_n);
        unsigned sa = (unsigned)__cvta_generic_to_shared(&stage[warp][lane][(f & 3) * 2]);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(src) : "memory");
      }
      asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
      acc += stage[warp][lane][0];
    } else {
      for (int f = 0; f < inflight; ++f)
        acc += __ldg(big + ((pos + (size_t)f * 64 + lane * 2) % big_n));
    }
    if (mode == 3)
      acc += (double)ldr(myword);
    pos += nw * 64 * inflight;
  }
  if (lane == 0)
    atomicAdd(out + 1, rounds * (unsigned long long)inflight * 512ull);
  if (acc == 12345.0)
    sink[0] = acc;
}

int main() {
  const size_t big_n = (size_t)1 << 30; // 8 GB of doubles
  double* big;
  cudaMalloc(&big, big_n * sizeof(double));
  cudaMemset(big, 0, big_n * sizeof(double));
  unsigned long long *words, *out;
  cudaMalloc(&words, (1 << 23) * 8);
  cudaMalloc(&out, 64);
  int* stop;
  cudaMalloc(&stop, 4);
  double* sink;
  cudaMalloc(&sink, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 50000;
  for (int mode : {0, 1, 4, 5})
    for (int inflight : {1, 4, 8}) {
      if ((mode == 0 || mode == 4) && inflight > 1)
        continue;
      for (int peer : {1, 150}) {
        cudaMemset(words, 0, (1 << 23) * 8);
        cudaMemset(stop, 0, 4);
        cudaMemset(out, 0, 64);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        k_hop<<<sms * 2, 256>>>(iters, peer, mode, inflight, words, big, big_n, stop, out, sink);
        cudaEventRecord(e1);
        cudaError_t e = cudaDeviceSynchronize();
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long h[2] = {0, 0};
        cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
        printf("mode=%d inflight=%d peer=%3d hop=%.1f ns  background %.0f GB/s (%s)\n", mode, inflight, peer,
               (double)h[0] / (2.0 * iters), (double)h[1] / (double)h[0], cudaGetErrorString(e));
      }
    }
  return 0;
}
