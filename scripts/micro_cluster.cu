// Microbenchmark: how many clusters of 8 / 16 CTAs are co-resident on this
// B200, and what one level of a cluster-synchronised level-set costs
// (store -> barrier.cluster release/acquire -> dependent L2 load).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o micro_cluster micro_cluster.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void cluster_sync_ra() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void k_levels(double* buf, int iters, int csize, unsigned long long* out) {
  const unsigned cr = cluster_rank();
  const int cl = blockIdx.x / csize;
  double* b = buf + (size_t)cl * csize * blockDim.x * 2;
  double acc = threadIdx.x;
  unsigned long long t0 = gtimer();
  for (int it = 0; it < iters; ++it) {
    double* w = b + (it & 1) * csize * blockDim.x;
    __stcg(w + cr * blockDim.x + threadIdx.x, acc);
    cluster_sync_ra();
    // read a word another CTA of the cluster wrote
    const unsigned src = (cr + 1 + (it % (csize - 1))) % csize;
    acc = __ldcg(w + src * blockDim.x + (threadIdx.x * 7 + it) % blockDim.x) * 0.5 + 1.0;
  }
  unsigned long long t1 = gtimer();
  if (threadIdx.x == 0)
    out[blockIdx.x] = t1 - t0;
  if (acc == -1.0)
    b[0] = acc;
}

__global__ void k_plain(double* buf, int iters, int csize, unsigned long long* out) {
  const unsigned cr = cluster_rank();
  unsigned long long t0 = gtimer();
  for (int it = 0; it < iters; ++it)
    cluster_sync_ra();
  unsigned long long t1 = gtimer();
  if (threadIdx.x == 0)
    out[blockIdx.x] = t1 - t0;
  if (cr == 1000)
    buf[0] = 1;
}

// DSMEM ping-pong: CTA 0 and CTA `peer` of a cluster bounce a counter through
// each other's shared memory (st.relaxed.cluster to the remote CTA, poll of
// the local word).  One hop = T / (2 iters).
__global__ void k_pingpong(int iters, int peer, unsigned long long* out) {
  __shared__ unsigned long long box;
  const unsigned cr = cluster_rank();
  if (threadIdx.x == 0)
    box = 0;
  cluster_sync_ra();
  unsigned long long t0 = gtimer();
  if (threadIdx.x == 0 && (cr == 0 || cr == (unsigned)peer)) {
    const unsigned other = cr == 0 ? peer : 0;
    unsigned la = (unsigned)__cvta_generic_to_shared(&box), ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(other));
    for (unsigned long long it = 1; it <= (unsigned long long)iters; ++it) {
      if (cr == 0) {
        asm volatile("st.relaxed.cluster.shared::cluster.u64 [%0], %1;" ::"r"(ra), "l"(2 * it - 1) : "memory");
        unsigned long long v;
        do asm volatile("ld.relaxed.cluster.shared::cta.u64 %0, [%1];" : "=l"(v) : "r"(la) : "memory");
        while (v != 2 * it);
      } else {
        unsigned long long v;
        do asm volatile("ld.relaxed.cluster.shared::cta.u64 %0, [%1];" : "=l"(v) : "r"(la) : "memory");
        while (v != 2 * it - 1);
        asm volatile("st.relaxed.cluster.shared::cluster.u64 [%0], %1;" ::"r"(ra), "l"(2 * it) : "memory");
      }
    }
  }
  unsigned long long t1 = gtimer();
  if (threadIdx.x == 0)
    out[blockIdx.x] = t1 - t0;
  cluster_sync_ra();
}

// Global-memory ping-pong between two CTAs (same cluster launch, so the
// placement is comparable): relaxed gpu-scope store / poll.
__global__ void k_pingpong_g(int iters, int peer, unsigned long long* words, unsigned long long* out) {
  const unsigned cr = cluster_rank();
  unsigned long long t0 = gtimer();
  if (threadIdx.x == 0 && blockIdx.x < 16 && (cr == 0 || cr == (unsigned)peer)) {
    unsigned long long* mine = words + (cr == 0 ? 0 : 32);
    unsigned long long* other = words + (cr == 0 ? 32 : 0);
    for (unsigned long long it = 1; it <= (unsigned long long)iters; ++it) {
      if (cr == 0) {
        asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(other), "l"(2 * it - 1) : "memory");
        unsigned long long v;
        do asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(mine) : "memory");
        while (v != 2 * it);
      } else {
        unsigned long long v;
        do asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(mine) : "memory");
        while (v != 2 * it - 1);
        asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(other), "l"(2 * it) : "memory");
      }
    }
  }
  unsigned long long t1 = gtimer();
  if (threadIdx.x == 0)
    out[blockIdx.x] = t1 - t0;
}

int main() {
  int threads = 512;
  size_t smem = 160 * 1024;
  for (int csize : {8, 16}) {
    for (auto kern : {k_levels, k_plain}) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = csize;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.gridDim = dim3(csize * 8);
    int nclusters = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&nclusters, (void*)k_levels, &cfg);
    printf("cluster %d: max active clusters = %d (%s)\n", csize, nclusters, cudaGetErrorString(e));
    if (nclusters < 1)
      continue;
    int ncl = nclusters < 8 ? nclusters : 8;
    cfg.gridDim = dim3(csize * ncl);
    double* buf;
    unsigned long long* out;
    cudaMalloc(&buf, (size_t)ncl * csize * threads * 2 * sizeof(double));
    cudaMemset(buf, 0, (size_t)ncl * csize * threads * 2 * sizeof(double));
    cudaMalloc(&out, 4096 * 8);
    const int iters = 20000;
    for (int rep = 0; rep < 2; ++rep) {
      e = cudaLaunchKernelEx(&cfg, k_levels, buf, iters, csize, out);
      cudaDeviceSynchronize();
      unsigned long long h[4096];
      cudaMemcpy(h, out, csize * ncl * 8, cudaMemcpyDeviceToHost);
      unsigned long long mx = 0;
      for (int i = 0; i < csize * ncl; ++i)
        mx = h[i] > mx ? h[i] : mx;
      printf("  %d clusters x %d: store+sync+ld level = %.1f ns (%s)\n", ncl, csize, (double)mx / iters,
             cudaGetErrorString(e));
      e = cudaLaunchKernelEx(&cfg, k_plain, buf, iters, csize, out);
      cudaDeviceSynchronize();
      cudaMemcpy(h, out, csize * ncl * 8, cudaMemcpyDeviceToHost);
      mx = 0;
      for (int i = 0; i < csize * ncl; ++i)
        mx = h[i] > mx ? h[i] : mx;
      printf("  %d clusters x %d: bare cluster barrier = %.1f ns (%s)\n", ncl, csize, (double)mx / iters,
             cudaGetErrorString(e));
    }
    cudaFree(buf);
    cudaFree(out);
  }
  {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 8;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.blockDim = dim3(32);
    cfg.gridDim = dim3(8);
    unsigned long long *out, *words;
    cudaMalloc(&out, 4096 * 8);
    cudaMalloc(&words, 4096 * 8);
    const int iters = 100000;
    for (int peer = 1; peer < 8; peer += 3) {
      cudaMemset(words, 0, 4096 * 8);
      cudaError_t e = cudaLaunchKernelEx(&cfg, k_pingpong, iters, peer, out);
      cudaDeviceSynchronize();
      unsigned long long h[8];
      cudaMemcpy(h, out, 64, cudaMemcpyDeviceToHost);
      printf("DSMEM hop (peer %d): %.1f ns (%s)\n", peer, (double)h[0] / (2.0 * iters), cudaGetErrorString(e));
      e = cudaLaunchKernelEx(&cfg, k_pingpong_g, iters, peer, words, out);
      cudaDeviceSynchronize();
      cudaMemcpy(h, out, 64, cudaMemcpyDeviceToHost);
      printf("global hop (peer %d): %.1f ns (%s)\n", peer, (double)h[0] / (2.0 * iters), cudaGetErrorString(e));
    }
  }
  return 0;
}
