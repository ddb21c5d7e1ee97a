// micro_fp64.cu -- single-warp dependent-latency probes on this GPU:
// DADD, DMUL, DFMA chains, the Markstein division step and a shared-memory
// load->use chain (cycles per link).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void probe(double* out, long long* cyc, int n) {
  double a = out[0], b = out[1];
  __shared__ double sm[64];
  sm[threadIdx.x] = a;
  __syncwarp();
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k)
      a = __dadd_rn(a, b);
  }
  long long t1 = clock64();
#pragma unroll 1
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k)
      a = __dmul_rn(a, b);
  }
  long long t2 = clock64();
#pragma unroll 1
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k)
      a = __fma_rn(a, b, 0.5);
  }
  long long t3 = clock64();
  int idx = threadIdx.x;
#pragma unroll 1
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k)
      idx = (int)sm[idx & 31] & 31;
  }
  long long t4 = clock64();
  // dsub(dmul) pairs, as in the row sums
  double acc = a;
#pragma unroll 1
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k)
      acc = __dsub_rn(acc, __dmul_rn(b, acc));
  }
  long long t5 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
    cyc[2] = t3 - t2;
    cyc[3] = t4 - t3;
    cyc[4] = t5 - t4;
  }
  out[2 + threadIdx.x] = a + idx + acc;
}

int main() {
  double* d;
  long long* c;
  cudaMalloc(&d, 64 * sizeof(double));
  cudaMalloc(&c, 8 * sizeof(long long));
  double h[2] = {1.0000001, 1e-9};
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  const int n = 1000;
  for (int rep = 0; rep < 2; ++rep)
    probe<<<1, 32>>>(d, c, n);
  long long hc[5];
  cudaMemcpy(hc, c, sizeof(hc), cudaMemcpyDeviceToHost);
  const char* names[5] = {"DADD", "DMUL", "DFMA", "LDS->use", "DSUB(DMUL)"};
  for (int k = 0; k < 5; ++k)
    printf("%-12s %.1f cycles per dependent link\n", names[k], (double)hc[k] / (16.0 * n));
  return 0;
}
